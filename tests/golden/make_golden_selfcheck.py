"""Verdicts of the REAL reference's embedded suite (itq3.run_selfcheck) -> tests/golden/selfcheck_ref.json.

    python tests/golden/make_golden_selfcheck.py
"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    import itq3

    res = [{"name": r.name, "passed": bool(r.passed), "detail": r.detail} for r in itq3.run_selfcheck()]
    json.dump(res, open(os.path.join(HERE, "selfcheck_ref.json"), "w"), indent=1)
    for r in res:
        print(r)


if __name__ == "__main__":
    main()
