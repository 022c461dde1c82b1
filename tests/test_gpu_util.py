"""GPU: the block utilities of the reference API (quantizer.py:78-197, transform.py:99-197) against
fixtures produced by the real reference (tests/golden/make_golden_util.py): bit-exact except the
excess kurtosis (numpy's ** 4 is libm pow; ours is a once-rounded fourth power) and the dense
Hadamard oracle (a GEMM whose summation order is not pinned)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2603_27914_b200")

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "util_cases.npz"))
LENGTHS = [1, 2, 5, 7, 8, 9, 16, 31, 100, 128, 129, 135, 256, 300, 1000, 1024, 4097]


@pytest.mark.parametrize("n", LENGTHS + ["const"])
def test_block_stats(n):
    s = P.block_stats(G[f"bs_in_{n}"])
    want = G[f"bs_out_{n}"]
    got = np.array([s.n, s.mean, s.sigma, s.l1, s.linf])
    np.testing.assert_array_equal(got, want[:5])  # pairwise sums, division, sqrt: bit-exact
    np.testing.assert_allclose(s.excess_kurtosis, want[5], rtol=1e-14, atol=1e-14)


def test_ternary_quantize_dequantize():
    x = G["tq_in"]
    for d, z in ((0.5, 0), (0.37, 1), (1.3, -1)):
        g = P.TernaryGrid(d=d, z=z)
        c = P.ternary_quantize(x, g)
        assert c.dtype == np.int8
        np.testing.assert_array_equal(c, G[f"tq_{d}_{z}"])
        np.testing.assert_array_equal(P.ternary_dequantize(c, g), G[f"td_{d}_{z}"])
    assert P.ternary_quantize(0.75, P.TernaryGrid(d=0.5)) == 1  # 1.5 -> 2 -> clipped
    assert isinstance(P.ternary_dequantize(1, P.TernaryGrid(d=0.5)), float)
    with pytest.raises(P.DomainError):
        P.ternary_quantize(np.array([1.0, np.nan]), P.TernaryGrid(d=0.5))
    with pytest.raises(P.DomainError):
        P.ternary_dequantize(np.array([2]), P.TernaryGrid(d=0.5))


def test_uniform_quantize():
    x = G["tq_in"]
    for bits, lo, hi in ((2, -1.0, 1.0), (3, -2.5, 1.5), (8, -0.7, 0.9)):
        np.testing.assert_array_equal(P.uniform_quantize(x, bits, lo, hi), G[f"uq_{bits}"])
    with pytest.raises(P.DomainError):
        P.uniform_quantize(x, 9, -1.0, 1.0)


def test_hadamard_and_staged_transforms():
    for n in (2, 4, 8, 16, 32, 64):
        np.testing.assert_array_equal(P.hadamard_matrix(n), G[f"hm_{n}"])
        np.testing.assert_allclose(P.hadamard_oracle(G[f"ho_in_{n}"]), G[f"ho_out_{n}"], rtol=1e-13, atol=1e-13)
    with pytest.raises(P.LengthError):
        P.hadamard_matrix(128)
    for n in (2, 8, 32, 256, 512):
        for dt in ("float64", "float32"):
            key = f"fs_{n}_{dt}"
            tr = P.fwht_staged(G[key + "_in"])
            assert tr.stage_count == int(np.log2(n))
            np.testing.assert_array_equal(np.stack(tr.stages), G[key + "_stages"])
            np.testing.assert_array_equal(tr.final, G[key + "_final"])
            assert tr.final.dtype == np.dtype(dt)
    np.testing.assert_array_equal(P.fwht32_warp(G["fw_in"]), G["fw_out"])
    with pytest.raises(P.LengthError):
        P.fwht32_warp(np.zeros(16))
