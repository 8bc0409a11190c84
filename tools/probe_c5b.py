import sys, time
import torch
sys.path.insert(0, ".")
import paper_2410_19208_b200 as psd
from oracle import sdls_oracle as so
prob = so.config5_instance(4096, 20000, nnz_per=4, seed=5)
beta = so.lipschitz_beta(prob)
sp = psd.SparseSdlsProblem(prob.c, 1.0, prob.con, prob.rows, prob.cols, prob.vals, prob.b)
cfg = psd.ProjectorConfig(method="randomized", params=psd.RangeParams(k=64, l=10, q=1))
psd.solve(sp, cfg, beta=beta, epsilon=1e-300, max_iter=3, rng=psd.DeviceRng(1))
torch.cuda.synchronize()
for its in (10, 110):
    t0 = time.perf_counter()
    psd.solve(sp, cfg, beta=beta, epsilon=1e-300, max_iter=its, rng=psd.DeviceRng(2))
    torch.cuda.synchronize()
    print(its, time.perf_counter() - t0, flush=True)
