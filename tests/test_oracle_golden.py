"""Pin the CPU oracle (oracle/itq3_oracle.py) to the reference's own outputs.

The fixtures were produced by tests/golden/make_golden.py running the real reference
package; here the oracle must reproduce them bit for bit (bytes, dequant values) and to
~1e-12 for the float64 fused products (the reference accumulates block by block).
"""

import hashlib
import os

import numpy as np
import pytest

from cases import case_inputs
from oracle import itq3_oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_small_cases_bit_exact(golden):
    meta, arrays, _ = golden
    assert len(meta) >= 200
    for i, c in enumerate(meta):
        w, x, X = case_inputs(i, tuple(c["shape"]), c["dist"])
        assert sha(w) == c["w_sha256"], f"{c['key']}: numpy generator drift"
        rows, cols = w.shape
        n, ss = c["block_n"], c["variant"] == "ss"
        pay, pad = O.quantize_payload(w, n, c["variant"], c["symmetric"], c["policy"])
        data = O.container_bytes(pay, rows, cols, n, c["variant"], c["symmetric"], pad)
        assert data == arrays[c["key"] + "_container"].tobytes(), c["key"]
        deq = O.dequantize(pay, rows, cols, n, ss)
        assert sha(deq) == c["deq_sha256"], c["key"]
        assert sha(np.signbit(deq)) == c["deq_signbit_sha256"], c["key"]
        y = O.fused_matmul(pay, rows, cols, n, ss, x[:, None])[:, 0]
        np.testing.assert_allclose(y, arrays[c["key"] + "_y"], rtol=1e-9, atol=1e-9)
        Y = O.fused_matmul(pay, rows, cols, n, ss, X)
        np.testing.assert_allclose(Y, arrays[c["key"] + "_Y"], rtol=1e-9, atol=1e-9)


def test_known_answer_vectors():
    # test_packing.py:24-35, 128-131 and test_transform.py:19-37 of the reference
    assert O.pack_planes(np.zeros((1, 256), np.int8)).tobytes() == b"\xff" * 32 + b"\x00" * 64
    assert O.pack_planes(np.full((1, 256), -1, np.int8)).tobytes() == b"\x00" * 96
    assert O.pack_planes(np.array([[-1, 0, 1, 1, 0, -1, 0, 0]], np.int8)).tobytes() == bytes([0xD2, 0x0C, 0x00])
    blk = O.serialize(np.array([[-1, 0, 1, 1, 0, -1, 0, 0]], np.int8), O.f16_bits([1.0]), O.f16_bits([0.0]))
    assert blk.tobytes() == bytes([0xD2, 0x0C, 0x00, 0x00, 0x3C, 0x00, 0x00])
    np.testing.assert_array_equal(O.fwht(np.array([1.0, 2.0, 3.0, 4.0])), [5.0, -1.0, -2.0, 0.0])
    v = np.zeros(256)
    v[37] = 7.5
    np.testing.assert_array_equal(np.abs(O.fwht(v)), np.full(256, 7.5 / 16.0))
    assert O.f16_bits(1e6)[()] == 0x7BFF and O.f16_bits(2049.0)[()] == 0x6800
    assert O.argmin_coeff().hex() == "0x1.c189374bc6a7fp-1"


def test_golden_containers():
    # test_golden.py:18-48: zero and impulse containers at n=32
    pay, pad = O.quantize_payload(np.zeros((1, 32)), 32)
    assert O.container_bytes(pay, 1, 32, 32, "s", True, pad)[32:] == b"\xff" * 4 + b"\x00" * 8 + b"\x00" * 4
    w = np.zeros((1, 32))
    w[0, 1] = 16.0
    pay, pad = O.quantize_payload(w, 32)
    assert pay.tobytes() == b"\x00" * 4 + b"\x55" * 4 + b"\x00" * 4 + b"\x83\x40" + b"\x00\x00"
    out = O.dequantize(pay, 1, 32, 32, False)
    assert abs(out[0, 1] - 2.255859375 * np.sqrt(32.0)) < 1e-12


@pytest.mark.slow
def test_full_c1_digests(golden):
    _, _, full = golden
    for c in full["c1"][:2]:
        w = O.generate_weights(c["dist"], 4096, 4096, seed=0).astype(np.float32)
        assert sha(w) == full["inputs"][f"{c['dist']}_4096x4096_seed0_f32"]
        pay, pad = O.quantize_payload(w, 256, c["variant"], c["symmetric"])
        data = O.container_bytes(pay, 4096, 4096, 256, c["variant"], c["symmetric"], pad)
        assert hashlib.sha256(data).hexdigest() == c["container_sha256"]
        deq = O.dequantize(pay, 4096, 4096, 256, c["variant"] == "ss")
        assert sha(deq) == c["dequant_f64_sha256"]
        err = O.eval_error(w, pay, 256, c["variant"] == "ss")
        assert err["mse"] == pytest.approx(c["mse"], rel=1e-12)
        assert err["frobenius_rel"] == pytest.approx(c["frobenius_rel"], rel=1e-12)


# --- evaluation harness (compute.py:136-400) pinned to tests/golden/eval_cases.json -------------
def _eval_golden():
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "eval_cases.json")) as f:
        return json.load(f)


def _eval_inputs(case):
    dist, rows, cols, seed, scale = case[:5]
    return O.generate_weights(dist, rows, cols, seed) * scale


def _cmp_report(got: dict, want: dict, where: str):
    """Exact equality for every field; frobenius_rel to rounding (BLAS ddot order)."""
    for k, v in want.items():
        ref = float.fromhex(v) if isinstance(v, str) else v
        if k == "frobenius_rel":
            assert got[k] == pytest.approx(ref, rel=1e-13, abs=0.0), (where, k)
        elif isinstance(ref, float) and np.isnan(ref):
            assert np.isnan(got[k]), (where, k)
        else:
            assert got[k] == ref, (where, k, got[k], ref)


@pytest.mark.parametrize("i", range(11))
def test_oracle_eval_reports(i):
    g = _eval_golden()["cases"][i]
    case = g["case"]
    w = _eval_inputs(case)
    n, variant, sym, kind = case[5:]
    calls = {"eval_error": lambda: O.error_report(w, n, variant, sym, kind),
             "eval_container": lambda: O.container_report(w, O.quantize_payload(w, n, variant, sym, kind)[0], n,
                                                          variant, sym, kind),
             "rotation_benefit": lambda: O.rotation_benefit(w, n, variant, sym, kind)}
    for key, fn in calls.items():
        want = g[key]
        if "raises" in want:
            with pytest.raises(O.NonFiniteError, match=want["message"]):
                with np.errstate(all="ignore"):
                    fn()
        else:
            with np.errstate(all="ignore"):
                _cmp_report(fn(), want, f"{case}:{key}")


def test_oracle_pairwise_sum_matches_numpy():
    rng = np.random.default_rng(5)
    for n in (1, 7, 8, 100, 128, 129, 1000, 4099, 65536 + 13):
        v = rng.standard_normal(n) ** 2
        assert O.pairwise_sum(v) == np.sum(v), n


def test_scalar_rules_vs_reference_fixtures():
    """ternary_mse (closed form vs the reference's quadrature) and optimal_scale, host scalars."""
    import paper_2603_27914_b200 as P

    G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "util_cases.npz"))
    for alpha, sigma, want in G["mse"]:
        assert abs(P.ternary_mse(alpha, sigma) - want) <= 1e-10 + 1e-9 * abs(want)
    s = G["os_stats"]
    st = P.BlockStats(n=int(s[0]), mean=s[1], sigma=s[2], l1=s[3], linf=s[4], excess_kurtosis=s[5])
    got = [P.optimal_scale(st, P.ScalePolicy(kind=k)) for k in ("constant", "argmin", "mean-abs")]
    np.testing.assert_array_equal(got, G["os_out"])


@pytest.mark.slow
def test_c3_samples_oracle(golden):
    """The oracle's fused_matmul reproduces the reference's C3 row samples (make_golden.py C3_EXTRA)."""
    _, _, full = golden
    here = os.path.join(os.path.dirname(__file__), "golden")
    for c in full["c3"][1:]:
        w = O.generate_weights("gaussian", c["rows"], c["cols"], seed=c["seed"]).astype(np.float32)
        X = np.random.default_rng(c["x_seed"]).standard_normal((c["cols"], c["m"])).astype(np.float32)
        assert sha(w) == c["input_sha256"] and sha(X) == c["x_sha256"]
        pay, pad = O.quantize_payload(w)
        data = O.container_bytes(pay, c["rows"], c["cols"], 256, "s", True, pad)
        assert hashlib.sha256(data).hexdigest() == c["container_sha256"]
        Y = O.fused_matmul(pay, c["rows"], c["cols"], 256, False, X)
        np.testing.assert_allclose(Y, np.load(os.path.join(here, c["y_file"])), rtol=1e-9, atol=1e-12)
