"""Kernel timeline (CUPTI through torch.profiler, chrome trace) of C3 projections with and
without the pipelined prefetch: per kernel its stream, start and duration, so the slow-down of the
main-stream kernels under the side stream's HBM traffic can be read kernel by kernel.
Usage: python tools/timeline_pf.py [n] → gpurun_out/tl/{pf,nopf}.json + a per-kernel table."""
import collections
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2410_19208_b200 as psd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
dev = torch.device("cuda", 0)
pool = [psd.workloads.c3_device(n, seed=s, device=dev) for s in range(2)]
params = psd.RangeParams(k=256, l=16, q=1)
rng = psd.DeviceRng(1)
out = torch.empty((n, n), dtype=torch.float64, device=dev)
os.makedirs("gpurun_out/tl", exist_ok=True)
from torch.profiler import ProfilerActivity, profile  # noqa: E402


def short(nm):
    return nm.split("(")[0].split("<")[0].split("::")[-1]


def run(tag, pf, reps=4):
    for i in range(3):
        psd.ran_proj(pool[i % 2], params, rng, out=out, prefetch=pool[(i + 1) % 2] if pf else None)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(reps):
            psd.ran_proj(pool[(i + 1) % 2], params, rng, out=out, prefetch=pool[i % 2] if pf else None)
        torch.cuda.synchronize()
    path = f"gpurun_out/tl/{tag}.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    main_stream = collections.Counter(e["args"]["stream"] for e in ev if "i8_gemm2" in e["name"]).most_common(1)[0][0]
    t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
    print(f"== {tag}: {(t1 - t0) / 1e3 / reps:.3f} ms per projection, {len(ev) / reps:.0f} kernels")
    tot = collections.defaultdict(lambda: [0.0, 0])
    for e in ev:
        key = (short(e["name"]), "main" if e["args"]["stream"] == main_stream else "side")
        tot[key][0] += e["dur"]
        tot[key][1] += 1
    for (nm, st), (us, c) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:28]:
        print(f"  {us / reps:9.1f} us  x{c / reps:5.1f}  avg {us / c:8.1f}  {st}  {nm}")
    # the third projection, kernel by kernel (main-stream idle gaps included)
    gemm_starts = [e["ts"] for e in ev if "philox" in e["name"]]
    if len(gemm_starts) >= 4:
        a, b = gemm_starts[2], gemm_starts[3]
        last_end = None
        for e in ev:
            if a <= e["ts"] < b:
                st = "M" if e["args"]["stream"] == main_stream else "s"
                gap = ""
                if st == "M":
                    if last_end is not None and e["ts"] - last_end > 3:
                        gap = f"   (main idle {e['ts'] - last_end:.0f} us before)"
                    last_end = e["ts"] + e["dur"]
                print(f"    {st} +{(e['ts'] - a) / 1e3:8.3f} ms  {e['dur']:8.1f} us  {short(e['name'])}{gap}")


run("nopf", False)
run("pf", True)
