"""Golden ErrorReports from the REAL reference evaluation harness (run in the build container).

    python tests/golden/make_golden_eval.py

Imports ``itq3`` from /root/reference/pkg/src (read-only) and writes tests/golden/eval_cases.json:
for every case of ``EVAL_CASES`` the reference's eval_error, eval_container (of its own
quantize_tensor output) and rotation_benefit, floats stored with float.hex so equality is exact.
Inputs are regenerated from (dist, rows, cols, seed, scale) with numpy's seeded generators.
"""

from __future__ import annotations

import json
import os
import sys
from dataclasses import asdict

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (dist, rows, cols, seed, scale, block_n, variant, symmetric, policy)
EVAL_CASES = [
    ("gaussian", 16, 512, 1, 1.0, 256, "s", True, "constant"),
    ("gaussian", 7, 300, 2, 1.0, 256, "s", True, "constant"),       # tail pad (2100 = 8*256 + 52)
    ("student-t", 32, 512, 41, 1.0, 256, "s", True, "constant"),
    ("outlier", 40, 512, 45, 1.0, 256, "s", False, "argmin"),
    ("laplace", 9, 448, 3, 1.0, 128, "ss", False, "mean-abs"),
    ("gaussian", 5, 1024, 4, 1.0, 512, "ss", True, "constant"),
    ("outlier", 12, 96, 5, 1.0, 32, "s", False, "constant"),
    ("student-t", 6, 200, 6, 1.0, 64, "ss", True, "argmin"),
    ("gaussian", 3, 512, 7, 0.0, 256, "s", True, "constant"),       # zero tensor
    ("gaussian", 4, 512, 8, 3.0e5, 256, "s", True, "constant"),     # f16 overflow: astype -> inf
    ("laplace", 64, 1024, 9, 1.0, 256, "s", False, "mean-abs"),
]


def inputs(dist, rows, cols, seed, scale):
    sys.path.insert(0, os.path.join(HERE, "..", ".."))
    from oracle.itq3_oracle import generate_weights

    return generate_weights(dist, rows, cols, seed) * scale


def hexd(d: dict) -> dict:
    return {k: (float(v).hex() if isinstance(v, float) else v) for k, v in d.items()}


def main():
    sys.path.insert(0, REF)
    import itq3
    from itq3.codec import QuantConfig
    from itq3.quantizer import ScalePolicy

    out = []
    for case in EVAL_CASES:
        dist, rows, cols, seed, scale, n, variant, sym, kind = case
        w = inputs(dist, rows, cols, seed, scale)
        assert np.array_equal(w, itq3.generate_weights(dist, rows, cols, seed) * scale)
        cfg = QuantConfig(block_n=n, variant=variant, symmetric=sym, policy=ScalePolicy(kind=kind))
        res = {"case": list(case)}
        q = itq3.quantize_tensor(w, cfg)
        for key, fn in (("eval_error", lambda: asdict(itq3.eval_error(w, cfg))),
                        ("eval_container", lambda: asdict(itq3.eval_container(w, q, ScalePolicy(kind=kind)))),
                        ("rotation_benefit", lambda: itq3.rotation_benefit(w, cfg))):
            try:
                with np.errstate(all="ignore"):
                    res[key] = hexd(fn())
            except itq3.ItqError as e:  # recorded: the product must raise the same class + message
                res[key] = {"raises": type(e).__name__, "message": str(e)}
        out.append(res)
    abl = itq3.ablate_block_size(sweep=(32, 64, 128, 256, 512), rows=4, cols=512, replicates=3)
    doc = {"cases": out, "ablate": [hexd(asdict(r)) for r in abl],
           "ablate_args": {"sweep": [32, 64, 128, 256, 512], "rows": 4, "cols": 512, "replicates": 3}}
    with open(os.path.join(HERE, "eval_cases.json"), "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", len(out), "cases")


if __name__ == "__main__":
    main()
