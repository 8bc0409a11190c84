"""Isolated launches of the INT8 reconstruction (psd_syrk_f64_int8, Ozaki-I
digit slices) at the C3 shape, next to the DMMA mirrored SYRK (psd_reconstruct),
for CUDA-event timing and ncu captures.

    python tools/probe_syrk.py [n] [r] [reps]
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_19208_b200 as psd  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    r = int(sys.argv[2]) if len(sys.argv) > 2 else 158
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    dev = torch.device("cuda", 0)
    lib = psd._native.load_library()
    nat = psd._native
    st = nat.stream_handle(dev)
    w = torch.linalg.qr(torch.randn(n, r, dtype=torch.float64, device=dev))[0].contiguous()
    d = torch.rand(r, dtype=torch.float64, device=dev) * 100 + 1
    c = torch.empty(n, n, dtype=torch.float64, device=dev)

    def t_int8():
        nat.check(lib.psd_syrk_f64_int8(nat.ptr(w), w.stride(0), nat.ptr(d), n, r, nat.ptr(c), n, st))

    def t_dmma():
        psd.symmetric.reconstruct_device(w, d, n, dev)

    for name, fn in (("int8", t_int8), ("dmma", t_dmma)):
        times = []
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        print(f"{name}: n={n} r={r} ms={sorted(times)} (includes scratch alloc / slices)", flush=True)
    ref = (w[:2048] * d) @ w.T
    t_int8()
    torch.cuda.synchronize()
    rel = (torch.linalg.norm(c[:2048] - ref) / torch.linalg.norm(ref)).item()
    print(f"rel err rows[:2048] {rel:.3e}; symmetric {torch.equal(c[:4096, :4096], c[:4096, :4096].T)}")


if __name__ == "__main__":
    main()
