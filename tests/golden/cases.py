"""Seeded small-case definitions shared by make_golden.py (reference side) and the tests.

Inputs are regenerated from these seeds on any box (numpy is the same in the image), so
the committed fixtures hold only the reference's OUTPUTS plus input digests.
"""

import numpy as np


def case_inputs(i: int, shape, dist: str):
    """Seeded inputs for small case i (same on every box)."""
    rng = np.random.default_rng(1000 + i)
    if dist == "gaussian":
        w = rng.standard_normal(shape)
    elif dist == "student-t":
        w = rng.standard_t(3, size=shape) * 10.0 ** rng.uniform(-3, 3)
    elif dist == "laplace":
        w = rng.laplace(size=shape)
    elif dist == "outlier":
        w = rng.standard_normal(shape)
        w.reshape(-1)[rng.integers(0, w.size, max(1, w.size // 100))] *= 20.0
    else:  # "edge": degenerate / extreme blocks (test_compute.py:117-129)
        h = np.where(np.array([bin(k & j).count("1") % 2 for k in range(256) for j in range(256)])
                     .reshape(256, 256) == 0, 1.0, -1.0)
        w = np.array([rng.normal(size=256), rng.laplace(size=256), rng.standard_t(3, size=256) * 1e4,
                      np.zeros(256), (h @ np.full(256, 3.0)) / 16.0])
    x = rng.standard_normal(w.shape[1])
    X = rng.standard_normal((w.shape[1], 3))
    return w, x, X


def case_list():
    shapes = [(1, 32), (3, 300), (4, 256), (2, 512), (5, 97), (8, 512), (16, 1024), (3, 1000)]
    cases = []
    i = 0
    for shape in shapes:
        for n in (32, 64, 128, 256, 512):
            for variant, sym, kind in (("s", True, "constant"), ("ss", True, "constant"),
                                       ("s", False, "constant"), ("s", True, "argmin"),
                                       ("ss", False, "mean-abs")):
                cases.append(dict(key=f"c{i:03d}", shape=list(shape), block_n=n, variant=variant,
                                  symmetric=sym, policy=kind, dist=["gaussian", "student-t", "laplace",
                                                                    "outlier"][i % 4]))
                i += 1
    for variant in ("s", "ss"):
        for sym in (True, False):
            cases.append(dict(key=f"c{i:03d}", shape=[5, 256], block_n=256, variant=variant, symmetric=sym,
                              policy="constant", dist="edge"))
            i += 1
    return cases


