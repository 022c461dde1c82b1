"""K8 evaluation harness (csrc/eval.cu via paper_2603_27914_b200.evaluate) vs the reference.

Golden: tests/golden/eval_cases.json (the real reference's eval_error / eval_container /
rotation_benefit / ablate_block_size, floats as hex) and full_digests.json (eval_error at C1,
4096x4096).  Every ErrorReport field must be EQUAL to the reference's; frobenius_rel (BLAS ddot
in the reference) to rel 1e-13.  Larger shapes are checked against the oracle the same way.
"""

import json
import math
import os

import numpy as np
import pytest
import torch

import paper_2603_27914_b200 as P
from oracle import itq3_oracle as O
from test_oracle_golden import _cmp_report, _eval_golden, _eval_inputs

pytestmark = pytest.mark.gpu


def cfg_of(case):
    n, variant, sym, kind = case[5:]
    return P.QuantConfig(block_n=n, variant=variant, symmetric=sym, policy=P.ScalePolicy(kind=kind))


@pytest.mark.parametrize("i", range(11))
def test_eval_matches_reference_golden(i):
    g = _eval_golden()["cases"][i]
    case = g["case"]
    w = _eval_inputs(case)
    cfg = cfg_of(case)
    q = P.quantize_tensor(w, cfg)
    calls = {"eval_error": lambda: vars(P.eval_error(w, cfg)),
             "eval_container": lambda: vars(P.eval_container(w, q, cfg.policy)),
             "rotation_benefit": lambda: P.rotation_benefit(w, cfg)}
    for key, fn in calls.items():
        want = g[key]
        if "raises" in want:
            with pytest.raises(getattr(P, want["raises"]), match=want["message"]):
                fn()
        else:
            _cmp_report(fn(), want, f"{case}:{key}")


def test_eval_c1_against_reference_digests(golden):
    _, _, full = golden
    for c in full["c1"][:3]:
        w = O.generate_weights(c["dist"], 4096, 4096, seed=0).astype(np.float32)
        r = P.eval_error(w, P.QuantConfig(variant=c["variant"], symmetric=c["symmetric"]))
        assert r.mse == c["mse"]
        assert r.zero_fraction == c["zero_fraction"]
        assert r.clamp_fraction == c["clamp_fraction"]
        assert r.frobenius_rel == pytest.approx(c["frobenius_rel"], rel=1e-13)
        assert r.n_blocks == 65536


@pytest.mark.parametrize("shape,n,variant,sym,kind,dist", [
    ((1024, 4096), 256, "s", True, "constant", "outlier"),
    ((333, 1000), 128, "ss", False, "argmin", "student-t"),
    ((2048, 1536), 512, "s", False, "mean-abs", "laplace"),
    ((100, 96), 32, "ss", True, "constant", "gaussian"),
])
def test_eval_matches_oracle_larger(shape, n, variant, sym, kind, dist):
    w = O.generate_weights(dist, *shape, seed=11)
    cfg = P.QuantConfig(block_n=n, variant=variant, symmetric=sym, policy=P.ScalePolicy(kind=kind))
    want = O.error_report(w, n, variant, sym, kind)
    _cmp_report(vars(P.eval_error(w, cfg)), want, "eval_error")
    # the same weights as a CUDA float64 tensor take the zero-copy path
    _cmp_report(vars(P.eval_error(torch.from_numpy(w).cuda(), cfg)), want, "eval_error(cuda)")
    q = P.quantize_tensor(w, cfg)
    pay = q.payload().cpu().numpy()
    _cmp_report(vars(P.eval_container(w, q, cfg.policy)), O.container_report(w, pay, n, variant, sym, kind),
                "eval_container")
    assert P.rotation_benefit(w, cfg) == O.rotation_benefit(w, n, variant, sym, kind)


def test_ablate_and_reports_match_reference():
    g = _eval_golden()
    a = g["ablate_args"]
    rows = P.ablate_block_size(sweep=tuple(a["sweep"]), rows=a["rows"], cols=a["cols"], replicates=a["replicates"])
    assert len(rows) == len(g["ablate"])
    for got, want in zip(rows, g["ablate"]):
        assert got.block_n == want["block_n"]
        assert got.mse == float.fromhex(want["mse"])
        assert got.relative_overhead == float.fromhex(want["relative_overhead"])
    data = json.loads(P.report_json(rows))
    assert [d["block_n"] for d in data] == a["sweep"]
    lines = P.report_csv(rows).strip().split("\n")
    assert lines[0] == "block_n,mse,relative_overhead" and len(lines) == 1 + len(rows)
    r = P.eval_error(P.generate_weights("gaussian", 4, 512, seed=47))
    assert set(json.loads(P.report_json(r))) == set(O.ERROR_FIELDS)
    assert P.report_csv(r).split("\n")[0] == ",".join(O.ERROR_FIELDS)


def test_eval_validation_and_edge_cases():
    with pytest.raises(P.ShapeError):
        P.eval_error(np.zeros(256))
    bad = np.zeros((2, 256))
    bad[0, 0] = np.inf
    with pytest.raises(P.DomainError, match="eval_error: input contains non-finite values"):
        P.eval_error(bad)
    r = P.eval_error(np.zeros((2, 512)))
    assert (r.mse, r.frobenius_rel, r.clamp_fraction, r.zero_fraction, r.bound_slack) == (0.0, 0.0, 0.0, 1.0, 0.0)
    # sign-pattern coefficients never clamp: the grid bound holds (test_compute.py:181-188)
    rng = np.random.default_rng(43)
    y = rng.choice([-1.0, 1.0], size=(4, 256)) * rng.uniform(0.95, 1.05, size=(4, 256))
    w = O.fwht(y).reshape(2, 512)
    r = P.eval_error(w)
    assert r.unclamped_blocks == 4 and r.bound_slack >= 0.0
    assert r.bound_slack == O.error_report(w)["bound_slack"]
    q = P.quantize_tensor(np.ones((2, 512)))
    with pytest.raises(P.ShapeError, match="does not match"):
        P.eval_container(np.ones((2, 256)), q)
    with pytest.raises(P.DomainError):
        P.ablate_block_size(sweep=(48,))
    with pytest.raises(P.DomainError):
        P.ablate_block_size(replicates=0)
    with pytest.raises(P.DomainError):
        P.generate_weights("cauchy", 2, 2, 0)


def test_eval_large_pairwise_tree():
    """235M-element-class reductions use the depth-capped node split; check a 6.3M tensor vs numpy."""
    w = O.generate_weights("gaussian", 3000, 2100, seed=3)  # 6.3M elements, ragged last block
    r = P.eval_error(w)
    want = O.error_report(w)
    _cmp_report(vars(r), want, "large")
    assert math.isfinite(r.mse)
