"""FP32 path vs FP64 path at full C3 size (n=32768, k=256, p=16, q=1) on the
same fp32-rounded X and Ω: the size-independent parity check for the FP32
path (the FP64 path is itself pinned to the oracle at 1e-10)."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2410_19208_b200 as psd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
dev = torch.device("cuda", 0)
x64 = psd.workloads.c3_device(n, seed=3, device=dev)
x32 = x64.float()
x64.copy_(x32)                       # the fp32-rounded X, upcast
g = torch.Generator(device=dev).manual_seed(5)
om = torch.randn(n, 272, device=dev, dtype=torch.float64, generator=g).float().double()
params = psd.RangeParams(k=256, l=16, q=1)
r64 = psd.ran_proj(x64, params, None, omega=om).result
del x64
torch.cuda.synchronize()
t = time.perf_counter()
rep = psd.ran_proj(x32, params, None, omega=om, dtype="fp32")
torch.cuda.synchronize()
r32 = rep.result
err = ((r32.double() - r64).norm() / r64.norm()).item()
print(f"n={n} KCHUNK={os.environ.get('PSD_TC32_KCHUNK', '0')}: fp32 vs fp64 rel frob {err:.3e} "
      f"(rank {rep.effective_rank}, {1e3 * (time.perf_counter() - t):.1f} ms incl. first-call setup)", flush=True)
