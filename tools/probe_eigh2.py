"""Device time of psd_eigh (CUDA events, 20 reps) and its sweep count, per m."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_19208_b200 as psd  # noqa: E402
from paper_2410_19208_b200 import _native  # noqa: E402

lib = _native.load_library()
for m in [int(x) for x in sys.argv[1:]] or [50, 74, 96, 144, 272]:
    rng = np.random.default_rng(0)
    q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    lam = np.concatenate([np.geomspace(1e3, 1, m // 2), -10 * rng.random(m - m // 2)])
    a = torch.from_numpy((q * lam) @ q.T).cuda()
    a = (a + a.T) / 2
    plan = _native.get_plan(m, m, a.device)
    vals = torch.empty(m, dtype=torch.float64, device="cuda")
    vecs = torch.empty((m, m), dtype=torch.float64, device="cuda")
    sw = ctypes.c_int32(0)
    ts = []
    for r in range(20):
        w = a.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.check(lib.psd_eigh(plan.handle, _native.ptr(w), m, m, _native.ptr(vals), _native.ptr(vecs), m,
                                   ctypes.byref(sw), _native.stream_handle(a.device)))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    err = np.abs(np.sort(vals.cpu().numpy()) - np.sort(lam)).max()
    print(f"m={m}: {np.median(ts)*1e3:.0f} us (min {min(ts)*1e3:.0f}), sweeps {sw.value}, eig err {err:.1e}", flush=True)
