"""Time the bench's FP32 leg call-by-call (device events + host wall) to find host gaps."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2410_19208_b200 as psd
from paper_2410_19208_b200 import workloads
n = 32768
dev = torch.device("cuda", 0)
params = psd.RangeParams(k=256, l=16, q=1)
pool = [workloads.c3_device(n, seed=i, device=dev) for i in range(2)]
pool32 = [x.float() for x in pool]
rng = psd.DeviceRng(seed=1)
for i in range(3):
    psd.ran_proj(pool32[i % 2], params, rng, dtype="fp32")
torch.cuda.synchronize()
for i in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    rep = psd.ran_proj(pool32[i % 2], params, rng, dtype="fp32")
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"call {i}: device {e0.elapsed_time(e1):.2f} ms, host {1e3*(t1-t0):.2f} ms, wall-after-sync {1e3*(time.perf_counter()-t0):.2f}", flush=True)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for i in range(3):
    rep = psd.ran_proj(pool32[i % 2], params, rng, dtype="fp32")
torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
