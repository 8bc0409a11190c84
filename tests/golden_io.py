"""Load the committed reference fixtures (tests/golden/*.npz) and regenerate
seeded inputs that were not stored verbatim."""

import glob
import os

import numpy as np

from oracle import psd_oracle as orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names(prefix=""):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, f"{prefix}*.npz")))


def load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    if "x" not in d and "x_kind" in d:
        kind = str(d["x_kind"])
        seed = int(d["x_seed"])
        if kind == "c1":
            d["x"] = orc.c1_matrix(seed=seed)
        elif kind == "wigner":
            n = int(d["n"]) if "n" in d else int(d["omega"].shape[0])
            d["x"] = orc.wigner(n, seed=seed)
        elif kind == "c3r40":
            d["x"] = orc.c3_matrix(int(d["omega"].shape[0]), seed=seed, rank=40)
        else:  # pragma: no cover
            raise KeyError(kind)
        if "x_checksum" in d:
            cs = np.array([float(np.sum(d["x"])), float(np.linalg.norm(d["x"]))])
            assert np.allclose(cs, d["x_checksum"], rtol=1e-12, atol=1e-12), \
                f"{name}: regenerated X drifted from the fixture (numpy RNG changed?)"
    return d


def golden_result(d):
    """Dense reference result, rebuilt from stored factors when not stored verbatim."""
    if "result" in d:
        return d["result"]
    w, dd = d["w"], d["d"]
    m = (w * dd) @ w.T
    return (m + m.T) / 2.0
