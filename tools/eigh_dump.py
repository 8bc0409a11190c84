"""Dump (or compare bit for bit) the device eigensolver's output on a fixed set of
matrices — a regression check for changes to the Jacobi kernel's scheduling that
must not change its arithmetic.  Usage: python tools/eigh_dump.py dump|cmp FILE"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2410_19208_b200 as psd  # noqa: E402

SIZES = [5, 20, 32, 33, 50, 64, 97, 144, 272, 300, 544]


def run():
    out = {}
    for m in SIZES:
        rng = np.random.default_rng(m)
        q, _ = np.linalg.qr(rng.standard_normal((m, m)))
        lam = np.concatenate([np.geomspace(1e3, 1, m // 2), -10 * rng.random(m - m // 2)])
        lam[: min(4, m)] = 7.0   # a repeated eigenvalue
        a = (q * lam) @ q.T
        a = (a + a.T) / 2
        vals, vecs = psd.symmetric.eigh_device(psd._tensors.as_device(torch.from_numpy(a).cuda()), validate=False)
        out[f"vals{m}"] = vals.cpu().numpy()
        out[f"vecs{m}"] = vecs.cpu().numpy()
        err = np.abs(np.sort(out[f"vals{m}"]) - np.sort(lam)).max() / np.abs(lam).max()
        print(f"m={m}: rel eig err {err:.2e}", flush=True)
    return out


def main():
    mode, path = sys.argv[1], sys.argv[2]
    out = run()
    if mode == "dump":
        np.savez(path, **out)
        return
    ref = np.load(path)
    bad = [k for k in out if not np.array_equal(out[k], ref[k])]
    print("bitwise identical" if not bad else f"DIFFER: {bad}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
