"""Compact summary of `ncu --set full` reports (read here, in the build container):
duration, SM clock, DRAM bytes, tensor-pipe activity, issue slots, occupancy and the
top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/ev/full_*.ncu-rep
"""
import csv
import io
import subprocess
import sys

UNIT = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
        "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
        "hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0}
KEYS = {
    "gpu__time_duration.sum": ("duration", None, "ms"),
    "sm__cycles_elapsed.avg.per_second": ("SM clock", None, "GHz"),
    "dram__bytes_read.sum": ("DRAM read", None, "GB"),
    "dram__bytes_write.sum": ("DRAM write", None, "GB"),
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": ("tensor pipe active", 1, "%"),
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": ("fp64 pipe", 1, "% of active"),
    "sm__inst_issued.avg.pct_of_peak_sustained_active": ("issue slots busy", 1, "%"),
    "sm__warps_active.avg.pct_of_peak_sustained_active": ("achieved occupancy", 1, "%"),
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": ("DRAM throughput", 1, "% of peak"),
    "launch__registers_per_thread": ("registers/thread", 1, ""),
    "launch__grid_size": ("grid", 1, "CTAs"),
}


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return f"{path}: no data"
    hdr, units, val = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, val))
    u = dict(zip(hdr, units))
    name = d.get("Kernel Name", "?")[:90]
    lines = [f"{name}"]
    for k, (label, scale, unit) in KEYS.items():
        if k in d and d[k] not in ("", "n/a"):
            try:
                sc = UNIT.get(u.get(k, ""), 1.0) if scale is None else scale
                v = float(d[k].replace(",", "")) * sc
                lines.append(f"  {label:22s} {v:10.3f} {unit}")
            except ValueError:
                pass
    pre = "smsp__pcsamp_warps_issue_stalled_"
    stalls = {k[len(pre):]: float(d[k] or 0) for k in hdr
              if k.startswith(pre) and not k.endswith("_not_issued") and d.get(k) not in ("", "n/a")}
    tot = sum(stalls.values())
    if tot > 0:
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
        lines.append("  top stall samples: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarize(p))
