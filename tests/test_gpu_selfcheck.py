"""GPU: the reference's embedded invariant suite (selfcheck.py) run against this package must give the
reference's own verdicts (tests/golden/selfcheck_ref.json, from make_golden_selfcheck.py): the same
fourteen named checks in order, the same pass/fail (the reference itself fails "ablation-trend"), and
the same detail line for the checks whose numbers are deterministic functions of the bit-exact codec."""

import json
import os

import pytest

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2603_27914_b200")

REF = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "selfcheck_ref.json")))
# detail lines that only involve exact codec values (float roundoff measurements differ by design)
SAME_DETAIL = {"outlier-bound", "grid-bound", "scale-oracle", "packing", "f16-codec", "rotation-benefit",
               "ablation-trend", "container-roundtrip"}


def test_run_selfcheck_matches_reference_verdicts():
    res = P.run_selfcheck()
    for r in res:
        print(f"{r.name:22s} {'PASS' if r.passed else 'FAIL'} {r.detail}")
    assert [r.name for r in res] == [x["name"] for x in REF]
    assert [r.passed for r in res] == [x["passed"] for x in REF]
    for r, x in zip(res, REF):
        if r.name in SAME_DETAIL:
            assert r.detail == x["detail"], (r.name, r.detail, x["detail"])
