"""Quick GPU probe: one C3-sized projection (n=32768, k=256, p=16, q=1) with
per-stage CUDA-event timings, plus the cuBLAS DGEMM rate for context.
Usage: python tools/probe_c3.py [n] [k] [p] [q]"""

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2410_19208_b200 as psd  # noqa: E402



def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    p = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    q = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    dtype = sys.argv[5] if len(sys.argv) > 5 else "fp64"
    dev = torch.device("cuda", 0)
    print(torch.cuda.get_device_name(0), flush=True)
    # cuBLAS DGEMM context number
    a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    b = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"cuBLAS DGEMM 8192^3: {2 * 8192**3 / best / 1e9:.1f} TFLOP/s", flush=True)
    del a, b
    t0 = time.time()
    x = psd.workloads.c3_device(n, seed=0, device=dev)
    torch.cuda.synchronize()
    if dtype == "fp32":
        x = x.float()
    print(f"generated X ({dtype}) in {time.time() - t0:.1f}s", flush=True)
    params = psd.RangeParams(k=k, l=p, q=q)
    rng = psd.DeviceRng(1)
    rep = psd.ran_proj(x, params, rng, assume_symmetric=False, dtype=dtype)
    plan = psd._native.get_plan(n, params.width, dev)
    plan.profile(enable=True, reset=True)
    for it in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = psd.ran_proj(x, params, rng, assume_symmetric=False, dtype=dtype)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        f = psd.flops(n, params, rep.effective_rank)
        print(f"proj {it}: {ms:.1f} ms  {f / ms / 1e9:.2f} TFLOP/s  r+={rep.effective_rank} "
              f"info={rep.device_info}", flush=True)
    prof = plan.profile(enable=False)
    for name, (ms, cnt) in prof.items():
        if cnt:
            print(f"  {name:12s} {ms / 3:9.2f} ms/proj  ({cnt // 3} marks/proj, {ms / cnt:.3f} ms each)")
    gm, gc = prof["sketch_gemm"]
    per = gm / gc
    print(f"sketch GEMM: {2 * n * n * params.width / per / 1e9:.2f} TFLOP/s per launch")


if __name__ == "__main__":
    main()
