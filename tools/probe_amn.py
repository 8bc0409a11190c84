import sys, torch
sys.path.insert(0, ".")
from paper_2410_19208_b200 import _native
lib = _native.load_library()
torch.set_printoptions(precision=3, linewidth=200)
def run(m, n, k, seed=0, show=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    at = torch.randn(k, m, device="cuda", generator=g)
    b = torch.randn(n, k, device="cuda", generator=g)
    c = torch.full((m, n), float("nan"), device="cuda", dtype=torch.float64)
    rc = lib.psd_gemm_tf32x3(2, _native.ptr(at), at.stride(0), _native.ptr(b), b.stride(0), m, n, k,
                             _native.ptr(c), c.stride(0), _native.stream_handle(at.device))
    torch.cuda.synchronize()
    ref = at.double().T @ b.double().T
    err = ((c - ref).norm() / ref.norm()).item()
    print(f"m={m} n={n} k={k} rc={rc} err={err:.3e}", flush=True)
    if show:
        print("c[:8,:4]", c[:8, :4]); print("ref[:8,:4]", ref[:8, :4])
        # try hypotheses
        for name, alt in [("A (not transposed, i.e. at as m x k)", None)]:
            pass
    return c, ref, at, b
c, ref, at, b = run(256, 32, 32, show=True)
# hypothesis checks on 256x32x32: compare c against products with permuted A
A = at.double().T  # m x k
for nm, Ap in [("k-rows permuted within 8", None)]:
    pass
print("rowerr", ((c - ref).abs().max(dim=1).values[:40]))
print("colerr", ((c - ref).abs().max(dim=0).values[:32]))
run(128, 16, 8); run(256, 16, 8); run(256, 16, 16); run(256, 16, 32); run(256,16,64); run(1024, 272, 4096)
