"""Stress the mirrored SYRK reconstruction: identical inputs, compare outputs bitwise."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2410_19208_b200 as psd
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
r = int(sys.argv[2]) if len(sys.argv) > 2 else 159
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
g = torch.Generator(device="cuda").manual_seed(1)
w = torch.randn(n, r + (r & 1), dtype=torch.float64, device="cuda", generator=g)[:, :r]   # even ld: TMA path
d = torch.rand(r, dtype=torch.float64, device="cuda", generator=g)
def recon(w, d):
    lib = psd._native.load_library()
    plan = psd._native.get_plan(n, r, torch.device("cuda"))
    out = torch.empty((n, n), dtype=torch.float64, device="cuda")
    psd._native.check(lib.psd_reconstruct(plan.handle, psd._native.ptr(w), n, w.stride(0),
                                          psd._native.ptr(d), r, psd._native.ptr(out), n,
                                          psd._native.stream_handle(torch.device("cuda"))))
    return out
ref = recon(w, d)
exact = (w * d) @ w.T
print("ld", w.stride(0))
bad = 0
for i in range(reps):
    out = recon(w, d)
    if not torch.equal(out, ref):
        bad += 1
        diff = (out != ref)
        idx = diff.nonzero()
        print(f"rep {i}: {int(diff.sum())} differing elements, first {idx[:3].tolist()}, "
              f"max |diff| {float((out-ref).abs().max()):.3e}", flush=True)
print("ref vs exact", float((ref - exact).abs().max() / exact.abs().max()), "symmetric", bool(torch.equal(ref, ref.T)))
print("BAD", bad, "of", reps)
