"""Config-5 solver loop timing: numpy Ω stream (reference order) vs device Philox."""
import cProfile, pstats, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2410_19208_b200 as psd
from oracle import sdls_oracle as so
prob = so.config5_instance(4096, 20000, nnz_per=4, seed=5)
beta = so.lipschitz_beta(prob)
sp = psd.SparseSdlsProblem(prob.c, 1.0, prob.con, prob.rows, prob.cols, prob.vals, prob.b)
cfg = psd.ProjectorConfig(method="randomized", params=psd.RangeParams(k=64, l=10, q=1))
psd.solve(sp, cfg, beta=beta, epsilon=1e-300, max_iter=3, rng=1)
torch.cuda.synchronize()
for label, rng in (("numpy", 1), ("device", psd.DeviceRng(7))):
    t0 = time.perf_counter()
    rep = psd.solve(sp, cfg, beta=beta, epsilon=1e-300, max_iter=30, rng=rng)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{label}: {30/dt:.1f} it/s ({1000*dt/30:.2f} ms/it)", flush=True)
plan = psd._native.get_plan(4096, 74, torch.device("cuda", 0))
plan.profile(enable=True, reset=True)
pr = cProfile.Profile(); pr.enable()
psd.solve(sp, cfg, beta=beta, epsilon=1e-300, max_iter=20, rng=1)
torch.cuda.synchronize()
pr.disable()
for k, (ms, c) in plan.profile(enable=False).items():
    if c: print(f"  {k:12s} {ms/20:.3f} ms/it ({c//20} marks)")
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
