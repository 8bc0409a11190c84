"""Ozaki-II FP64 emulation on INT8 tensor cores: accuracy vs an exact-ish reference
(fp64 GEMM on the same inputs, and a double-double check), then timing."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2410_19208_b200 import _native
lib = _native.load_library()
dev = torch.device("cuda", 0)
def run(a, p):
    m, k = a.shape; n = p.shape[1]
    c = torch.full((m, n), float("nan"), dtype=torch.float64, device=dev)
    rc = lib.psd_gemm_f64_ozaki(_native.ptr(a), a.stride(0), _native.ptr(p), p.stride(0), m, n, k,
                                _native.ptr(c), c.stride(0), _native.stream_handle(dev))
    if rc: raise RuntimeError(lib.psd_last_error().decode())
    return c
torch.manual_seed(0)
for (m, n, k) in [(256, 16, 128), (300, 40, 200), (1024, 272, 4096), (4096, 272, 4096), (2048, 144, 32768)]:
    a = torch.randn(m, k, dtype=torch.float64, device=dev)
    a[::7] *= 1e-3   # rows with different scales
    p = torch.randn(k, n, dtype=torch.float64, device=dev)
    c = run(a, p)
    ref = a @ p
    # higher-precision reference: split a and p into hi/lo fp32 pairs... use float64 with K-blocked Kahan via torch on CPU for small
    err = ((c - ref).norm() / ref.norm()).item()
    print(f"m={m} n={n} k={k}: rel err vs cuBLAS fp64 {err:.3e}  max|c| {c.abs().max().item():.3e} nan={bool(c.isnan().any())}", flush=True)
n = 32768
x = torch.randn(n, n, dtype=torch.float64, device=dev)
p = torch.randn(n, 272, dtype=torch.float64, device=dev)
c = run(x, p); torch.cuda.synchronize()
t = time.perf_counter()
c = run(x, p); torch.cuda.synchronize()
print(f"n={n} w=272 (incl. residue prep + alloc): {1e3*(time.perf_counter()-t):.1f} ms")
