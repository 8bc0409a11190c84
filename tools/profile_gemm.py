"""Isolated launches of the dominant kernel (op(X)·P DMMA GEMM at C3 shape)
for ncu captures and a CUDA-event timing of the same launch.

    python tools/profile_gemm.py [n] [w] [reps] [layout: nn|tn]
"""

import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_19208_b200 as psd  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    w = int(sys.argv[2]) if len(sys.argv) > 2 else 272
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    lay = sys.argv[4] if len(sys.argv) > 4 else "nn"
    dev = torch.device("cuda", 0)
    lib = psd._native.load_library()
    x = psd.workloads.c3_device(n, seed=1, device=dev)
    p = torch.randn(n, w, dtype=torch.float64, device=dev)
    c = torch.empty(n, w, dtype=torch.float64, device=dev)
    ws = torch.empty(4 * n * ((w + 1) // 2 * 2) + (1 << 20), dtype=torch.float64, device=dev)
    al = 1 if lay == "tn" else 0
    st = psd._native.stream_handle(dev)
    times = []
    for r in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        psd._native.check(lib.psd_gemm_f64(al, 0, psd._native.ptr(x), n, psd._native.ptr(p), w,
                                           psd._native.ptr(c), w, n, w, n, 0, 1.0,
                                           ctypes.c_void_p(0), 0, psd._native.ptr(ws), ws.numel(), st))
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ref = x[:4096] @ p
    err = ((c[:4096] - ref).abs().max() / ref.abs().max()).item()
    best = min(times[1:]) if len(times) > 1 else times[0]
    print(f"gemm {lay} n={n} w={w}: best {best:.3f} ms  {2 * n * n * w / best / 1e9:.2f} TFLOP/s "
          f"(times {[round(t, 3) for t in times]}) rel err {err:.2e}")


if __name__ == "__main__":
    main()
