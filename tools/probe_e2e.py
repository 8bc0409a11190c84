"""Timeline of ran_proj_many at C3: per-step upload / compute / download intervals (CUDA events)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2410_19208_b200 as psd
from paper_2410_19208_b200 import pipeline, workloads

dev = torch.device("cuda", 0)
n = 32768
params = psd.RangeParams(k=256, l=16, q=1)
hx = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
hx.copy_(workloads.c3_device(n, seed=1, device=dev).cpu())
hr = [torch.empty((n, n), dtype=torch.float64, pin_memory=True) for _ in range(2)]
rng = psd.DeviceRng(seed=7)

# monkeypatch torch.Tensor.copy_ timing via events around the pipeline's stream work
marks = []
orig_copy = torch.Tensor.copy_
def timed_copy(self, src, non_blocking=False):
    s = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s); r = orig_copy(self, src, non_blocking=non_blocking); e1.record(s)
    kind = "H2D" if src.device.type == "cpu" else ("D2H" if self.device.type == "cpu" else "D2D")
    marks.append((kind, e0, e1))
    return r
orig_run = psd.projection._run
def timed_run(*a, **k):
    s = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s); r = orig_run(*a, **k); e1.record(s)
    marks.append(("PROJ", e0, e1))
    return r
pipeline.ran_proj_many([hx], params, rng, out=[hr[0]])
torch.cuda.synchronize()
torch.Tensor.copy_ = timed_copy
psd.projection._run = timed_run
steps = 8
ref = torch.cuda.Event(enable_timing=True); ref.record()
t0 = time.perf_counter()
pipeline.ran_proj_many([hx] * steps, params, rng, out=[hr[i % 2] for i in range(steps)])
torch.cuda.synchronize()
wall = time.perf_counter() - t0
torch.Tensor.copy_ = orig_copy
merged = []
for kind, e0, e1 in marks:
    if merged and merged[-1][0] == kind and kind in ("H2D", "D2H") and abs(merged[-1][2].elapsed_time(e0)) < 5.0:
        merged[-1] = (kind, merged[-1][1], e1)
    else:
        merged.append((kind, e0, e1))
for kind, e0, e1 in merged:
    print(f"{kind:5s} {ref.elapsed_time(e0):9.1f} -> {ref.elapsed_time(e1):9.1f}  ({e0.elapsed_time(e1):7.1f} ms)")
print(f"wall {wall*1e3:.0f} ms for {steps} steps -> {steps/wall:.2f}/s")
