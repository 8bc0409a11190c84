"""Concurrent host threads on one device (the reference is 'safe for concurrent calls
with distinct Generators'): the library serializes calls per device, so
three threads on three streams neither deadlock (persistent TMEM kernels and the
cooperative eigensolver cannot share a GPU with copies of themselves) nor change any
result.  Run in a subprocess with a timeout so a regression fails instead of hanging."""

import os
import subprocess
import sys
import textwrap

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import sys, threading
    sys.path.insert(0, %r)
    import numpy as np, torch
    import paper_2410_19208_b200 as psd
    from oracle import psd_oracle as orc
    dev = torch.device("cuda", 0)
    n = 3584
    xs = [torch.from_numpy(orc.c3_matrix(n, seed=s, rank=48)).to(dev) for s in range(3)]
    oms = [torch.from_numpy(np.random.default_rng(10 + s).standard_normal((n, 72))).to(dev) for s in range(3)]
    prm = psd.RangeParams(k=64, l=8, q=1)
    seq = [psd.ran_proj(x, prm, None, omega=o).result.clone() for x, o in zip(xs, oms)]
    out = [None] * 3
    def work(i):
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            for _ in range(2):
                r = psd.ran_proj(xs[i], prm, None, omega=oms[i]).result
            s.synchronize()
            out[i] = r.clone()
    ts = [threading.Thread(target=work, args=(i,)) for i in range(3)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    torch.cuda.synchronize()
    ok = all(torch.equal(a, b) for a, b in zip(seq, out))
    print("CONCURRENT", "OK" if ok else "MISMATCH", flush=True)
""") % REPO


@pytest.mark.gpu
def test_three_threads_three_streams():
    res = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "CONCURRENT OK" in res.stdout
