"""GPU probe for the 3xTF32 tcgen05 GEMM: correctness vs fp64 torch, then timing."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2410_19208_b200 import _native  # noqa: E402

lib = _native.load_library()
dev = torch.device("cuda:0")


def gemm(mode, a, b, c):
    st = _native.stream_handle(dev)
    rc = lib.psd_gemm_tf32x3(mode, _native.ptr(a), a.stride(0), _native.ptr(b), b.stride(0),
                             a.shape[0], b.shape[0], a.shape[1], _native.ptr(c), c.stride(0), st)
    if rc != 0:
        raise RuntimeError(lib.psd_last_error().decode())


def check(m, n, k, mode=0, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    a = torch.randn(m, k, device=dev, generator=g, dtype=torch.float32)
    b = a if mode == 1 else torch.randn(n, k, device=dev, generator=g, dtype=torch.float32)
    if mode == 1:
        bb = torch.randn(n, k, device=dev, generator=g, dtype=torch.float32)
        b = bb
    ref = a.double() @ b.double().T
    if mode == 0:
        c = torch.full((m, n), float("nan"), device=dev, dtype=torch.float64)
        gemm(0, a, b, c)
        err = (c - ref).norm() / ref.norm()
    else:
        c = torch.full((m, m), float("nan"), device=dev, dtype=torch.float32)
        gemm(1, a, b, c)
        low = torch.tril(ref)
        refm = low + low.T - torch.diag(torch.diag(ref))
        err = (c.double() - refm).norm() / refm.norm()
        sym = bool((c == c.T).all())
        print(f"  mirror symmetric={sym}")
    torch.cuda.synchronize()
    print(f"mode={mode} m={m} n={n} k={k}: rel err {err.item():.3e}", flush=True)
    return err.item()


if __name__ == "__main__":
    errs = []
    for (m, n, k, mode) in [(128, 16, 16, 0), (128, 32, 64, 0), (256, 48, 64, 0), (1000, 272, 4096, 0),
                            (300, 520, 1000, 0), (512, 512, 40, 1), (1000, 1000, 64, 1)]:
        errs.append(check(m, n, k, mode))
    ok = all(e < 1e-5 for e in errs)
    print("ALL OK" if ok else "FAIL")
    if not ok:
        sys.exit(1)
    # timing: X·P at n=32768, w=272 via the C-ABI entry (includes its split + malloc)
    n, w = int(sys.argv[1]) if len(sys.argv) > 1 else 16384, 272
    a = torch.randn(n, n, device=dev, dtype=torch.float32)
    b = torch.randn(w, n, device=dev, dtype=torch.float32)
    c = torch.empty(n, w, device=dev, dtype=torch.float64)
    for _ in range(2):
        gemm(0, a, b, c)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        gemm(0, a, b, c)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"entry (split+gemm+alloc) n={n} w={w}: {dt*1e3:.2f} ms, {2*n*n*w/dt/1e12:.1f} TF/s effective")
