"""Kernel timeline of a few projections (CUPTI through torch.profiler): per-kernel
device time, and the GPU idle gaps between consecutive kernels — the cost of
host round trips and launch latency that per-kernel timings do not show.
Usage: python tools/timeline.py [c1|c2|c3] [reps]"""

import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2410_19208_b200 as psd  # noqa: E402

CFG = {"c1": (1000, 40, 10, 2), "c2": (8192, 128, 16, 2), "c3": (32768, 256, 16, 1)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    n, k, p, q = CFG[name]
    dev = torch.device("cuda", 0)
    x = psd.workloads.c3_device(n, seed=0, device=dev) if name == "c3" else psd.workloads.wigner_device(n, 0, dev)
    params = psd.RangeParams(k=k, l=p, q=q)
    rng = psd.DeviceRng(1)
    for _ in range(3):
        psd.ran_proj(x, params, rng, assume_symmetric=False)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            psd.ran_proj(x, params, rng, assume_symmetric=False)
        e1.record()
        torch.cuda.synchronize()
    wall = e0.elapsed_time(e1) / reps
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() >= 0]
    ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs
                if "Memcpy" not in e.name and "Memset" not in e.name)
    allops = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
    busy = collections.defaultdict(float)
    for s, t, nm in ks:
        busy[nm.split("(")[0].split("<")[0].split("::")[-1]] += (t - s)
    # idle = the union of all device activity subtracted from the span
    span0, span1 = allops[0][0], allops[-1][1]
    cover, cur_s, cur_t = 0.0, None, None
    gaps = []
    for s, t, nm in allops:
        if cur_t is None:
            cur_s, cur_t, last = s, t, nm
        elif s > cur_t:
            cover += cur_t - cur_s
            gaps.append((s - cur_t, last, nm))
            cur_s, cur_t = s, t
        else:
            cur_t = max(cur_t, t)
        last = nm if t >= cur_t else last
    cover += cur_t - cur_s
    span = span1 - span0
    print(f"{name}: {reps} projections, {wall:.3f} ms each (events); profiled span {span / 1e3 / reps:.3f} ms, "
          f"device busy {cover / 1e3 / reps:.3f} ms, idle {(span - cover) / 1e3 / reps:.3f} ms per projection")
    print(f"kernels per projection: {len(ks) / reps:.0f}, gaps > 2 us per projection: "
          f"{sum(1 for g in gaps if g[0] > 2) / reps:.1f}")
    print("per-projection device time by kernel (us):")
    for nm, us in sorted(busy.items(), key=lambda kv: -kv[1])[:20]:
        print(f"  {us / reps:10.1f}  {nm}")
    agg = collections.defaultdict(lambda: [0.0, 0])
    for g, a, b in gaps:
        key = (a.split("(")[0].split("<")[0].split("::")[-1][:28], b.split("(")[0].split("<")[0].split("::")[-1][:28])
        agg[key][0] += g
        agg[key][1] += 1
    print("largest idle gaps by (kernel before -> kernel after), us per projection:")
    for (a, b), (g, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:15]:
        print(f"  {g / reps:8.1f} us  x{c / reps:4.1f}  {a} -> {b}")


if __name__ == "__main__":
    main()
