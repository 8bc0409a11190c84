"""PCIe rates on the box: H2D, D2H alone and concurrently (pinned 8.6 GB buffers)."""
import time
import torch
n = 32768
dev = torch.device("cuda", 0)
h1 = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
h2 = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
d1 = torch.empty((n, n), dtype=torch.float64, device=dev)
d2 = torch.empty((n, n), dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
gb = 8 * n * n / 1e9
def t(fn):
    torch.cuda.synchronize(); a = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - a
for _ in range(2):
    th = t(lambda: d1.copy_(h1, non_blocking=True))
    td = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    tb = t(both)
    print(f"H2D {gb/th:.1f} GB/s  D2H {gb/td:.1f} GB/s  concurrent {2*gb/tb:.1f} GB/s total ({tb*1e3:.0f} ms for both)")
