import sys, torch
sys.path.insert(0, ".")
import paper_2410_19208_b200 as psd
from paper_2410_19208_b200 import workloads
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
mode = sys.argv[2] if len(sys.argv) > 2 else "omega"
dev = torch.device("cuda:0")
pool = [workloads.c3_device(n, seed=s, device=dev) for s in range(4)]
params = psd.RangeParams(k=256, l=16, q=1)
g = torch.Generator(device="cuda").manual_seed(3)
oms = [torch.randn((n, 272), dtype=torch.float64, device=dev, generator=g) for _ in range(6)]
refs = [psd.ran_proj(pool[i % 4], params, None, omega=oms[i]).result.clone() for i in range(6)]
out = torch.empty((n, n), dtype=torch.float64, device=dev)
rng = psd.DeviceRng(seed=1)
for i in range(6):
    nxt = pool[(i + 1) % 4] if i < 5 else None
    try:
        if mode == "omega":
            r = psd.ran_proj(pool[i % 4], params, None, omega=oms[i], out=out, prefetch=nxt)
            print(i, "equal", torch.equal(r.result, refs[i]), r.device_info["qr_passes"], flush=True)
        else:
            r = psd.ran_proj(pool[i % 4], params, rng, out=out, prefetch=nxt)
            print(i, "ok", r.effective_rank, r.device_info["qr_passes"], flush=True)
    except Exception as e:
        print(i, "ERR", e, flush=True)
