"""Does the tf32 tensor core truncate the low 13 mantissa bits? Compare 3xTF32
errors with rna-split operands vs raw-hi operands (run twice, env switch)."""
import os, sys
import torch
sys.path.insert(0, ".")
from paper_2410_19208_b200 import _native
lib = _native.load_library()
for (m, n, k) in [(256, 64, 64), (1000, 272, 4096), (2048, 272, 32768)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(m, k, device="cuda", generator=g)
    b = torch.randn(n, k, device="cuda", generator=g)
    c = torch.empty(m, n, device="cuda", dtype=torch.float64)
    _native.check(lib.psd_gemm_tf32x3(0, _native.ptr(a), k, _native.ptr(b), k, m, n, k, _native.ptr(c), n,
                                      _native.stream_handle(a.device)))
    ref = a.double() @ b.double().T
    f32 = (a @ b.T).double()
    print(f"RAWHI={os.environ.get('PSD_TF32_RAWHI','0')} m={m} n={n} k={k}: 3xtf32 err "
          f"{((c-ref).norm()/ref.norm()).item():.3e}  (torch fp32 matmul err {((f32-ref).norm()/ref.norm()).item():.3e})")
