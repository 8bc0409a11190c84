"""PCIe duplex rates on the box with and without a concurrent HBM-heavy kernel
load, and with the host buffers placed on the GPU's NUMA node (affinity set
before the pinned allocations).  Reports the host topology it sees.

    python tools/probe_pcie2.py [local|default]
"""
import glob
import os
import sys
import time

import torch

mode = sys.argv[1] if len(sys.argv) > 1 else "default"
dev = torch.device("cuda", 0)
props = torch.cuda.get_device_properties(dev)
bdf = None
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    bdf = pynvml.nvmlDeviceGetPciInfo(h).busId
    bdf = bdf.decode() if isinstance(bdf, bytes) else bdf
except Exception as exc:  # pragma: no cover
    print("nvml:", exc)
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
print("numa nodes:", [os.path.basename(n) for n in nodes], "cpus:", os.cpu_count())
local = None
if bdf:
    dom = bdf.lower()
    dom = dom[4:] if len(dom.split(":")[0]) == 8 else dom     # 00000000:xx:yy.z → 0000:xx:yy.z
    for path in (f"/sys/bus/pci/devices/{dom}", f"/sys/bus/pci/devices/{dom.lower()}"):
        if os.path.exists(path):
            try:
                local = open(f"{path}/local_cpulist").read().strip()
                node = open(f"{path}/numa_node").read().strip()
                print("gpu", dom, "numa_node", node, "local_cpulist", local)
            except OSError as exc:
                print("sysfs:", exc)
            break
if mode == "local" and local:
    cpus = set()
    for part in local.split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    os.sched_setaffinity(0, cpus)
    print("affinity ->", len(cpus), "cpus")

n = 32768
h1 = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
h2 = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
h1.fill_(1.0)
h2.fill_(2.0)
d1 = torch.empty((n, n), dtype=torch.float64, device=dev)
d2 = torch.empty((n, n), dtype=torch.float64, device=dev)
load_a = torch.empty((n, n), dtype=torch.float64, device=dev)
load_b = torch.empty((n, n), dtype=torch.float64, device=dev)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
gb = 8 * n * n / 1e9


def t(fn):
    torch.cuda.synchronize()
    a = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - a


def load(k):
    with torch.cuda.stream(s3):
        for _ in range(k):
            load_b.copy_(load_a)      # 17 GB of HBM traffic per copy


for rep in range(2):
    th = t(lambda: d1.copy_(h1, non_blocking=True))
    td = t(lambda: h2.copy_(d2, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    tb = t(both)

    def both_loaded():
        load(60)
        both()
    tl = t(both_loaded)

    def chunked():
        c = 8
        rows = n // c
        for j in range(c):
            with torch.cuda.stream(s1):
                d1[j * rows:(j + 1) * rows].copy_(h1[j * rows:(j + 1) * rows], non_blocking=True)
            with torch.cuda.stream(s2):
                h2[j * rows:(j + 1) * rows].copy_(d2[j * rows:(j + 1) * rows], non_blocking=True)
    tc = t(chunked)
    print(f"[{mode}] H2D {gb / th:.1f} GB/s  D2H {gb / td:.1f} GB/s  duplex {2 * gb / tb:.1f} GB/s "
          f"({tb * 1e3:.0f} ms)  duplex+HBM load {2 * gb / tl:.1f} GB/s ({tl * 1e3:.0f} ms, load alone "
          f"{t(lambda: load(60)) * 1e3:.0f} ms)  chunked duplex {2 * gb / tc:.1f} GB/s", flush=True)
