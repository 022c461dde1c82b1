"""GPU: K5 / K5b tcgen05 MMQ (csrc/mmq.cu) vs the exact fp64 product of the oracle-decoded weights.

fused_matmul sends 16 <= M <= 64 tokens to K5b (kind::i8, 16-bit fixed-point activations per
(token, block): test_gpu_stack.chain_bound at L = 2 per column) and M > 64 to K5 (kind::f16):

Tolerance: A = d*t is exact in f16, so the error comes only from the f16
rounding of the rotated activations x'' = H x / 16 (relative 2^-11 per element) and the fp32
butterfly / tensor-core accumulation:
    |err| <= sum_{b,k} |d t_k| (2^-10 |x''_k| + 2^-18 |x_b|_1 / 16) + 1e-5 sum |w_hat| |x|.
"""

import numpy as np
import pytest
import torch

from oracle import itq3_oracle as O

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2603_27914_b200")


def mmq_bound(payload, rows, cols, X, ss=False, n=256):
    nb = cols // n
    deq = O.dequantize(payload, rows, cols, n, ss)
    quants, sb, zb, sub = O.split_payload(payload, n, ss)
    codes, _ = O.unpack_planes(quants, n)
    t = codes.astype(np.float64) - np.trunc(O.f16_value(zb))[:, None]
    d = np.repeat(O.f16_value(sub), n // 8, axis=1) if ss else O.f16_value(sb)[:, None]
    a = np.abs(t * d).reshape(rows, cols)                                # |d t| per (row, k)
    Xd = np.asarray(X, np.float64)
    rs = 1.0 / np.sqrt(n)
    xr = O.butterfly(Xd.T.reshape(-1, nb, n)).reshape(-1, cols).T * rs   # x'' (cols x m)
    l1 = np.abs(Xd).reshape(nb, n, -1).sum(axis=1)                      # (nb, m)
    term = 2.0 ** -10 * np.abs(xr) + 2.0 ** -18 * np.repeat(l1, n, axis=0) * rs
    return deq @ Xd, a @ term + 1e-5 * (np.abs(deq) @ np.abs(Xd))


def matmul_bound(payload, rows, cols, X):
    """The a-priori bound of the path fused_matmul takes for X's token count (compute.py)."""
    m = X.shape[1]
    if P.compute.MMQ_MIN_TOKENS <= m <= P.compute.MMQ8_MAX_TOKENS:
        from test_gpu_stack import chain_bound

        cols_ = [chain_bound(payload, rows, cols, np.asarray(X, np.float64)[:, j], limbs=2) for j in range(m)]
        return np.stack([c[0] for c in cols_], axis=1), np.stack([c[1] for c in cols_], axis=1)
    return mmq_bound(payload, rows, cols, X)


@pytest.mark.parametrize("rows,cols", [(300, 512), (128, 1024), (1000, 256)])
@pytest.mark.parametrize("m", [8, 12, 16, 64, 100, 256, 300])
@pytest.mark.parametrize("asym", [False, True])
def test_mmq_matches_exact(rows, cols, m, asym):
    rng = np.random.default_rng(rows + cols + m)
    w = rng.standard_normal((rows, cols)) * 0.05
    q = P.quantize_tensor(w, P.QuantConfig(symmetric=not asym))
    X = rng.standard_normal((cols, m)).astype(np.float32)
    Y = P.fused_matmul(q, torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
    exact, bound = matmul_bound(q.payload().cpu().numpy(), rows, cols, X)
    assert np.all(np.abs(Y - exact) <= bound), np.max(np.abs(Y - exact) / bound)


def test_mmq_dtypes_and_strides():
    rng = np.random.default_rng(5)
    q = P.quantize_tensor(rng.standard_normal((256, 768)) * 0.1)
    X = torch.from_numpy(rng.standard_normal((768, 40)).astype(np.float32)).cuda()
    Y = P.fused_matmul(q, X)
    for dt in (torch.bfloat16, torch.float16):
        Yd = P.fused_matmul(q, X.to(dt)).cpu().numpy()
        exact, bound = matmul_bound(q.payload().cpu().numpy(), 256, 768, X.to(dt).float().cpu().numpy())
        assert np.all(np.abs(Yd - exact) <= bound)
    # token-major activations (M x K transposed view) -> identical result
    Y2 = P.fused_matmul(q, X.t().contiguous().t())
    torch.testing.assert_close(Y, Y2, rtol=0, atol=0)


@pytest.mark.parametrize("rows,cols,m", [(8192, 1024, 640), (4352, 512, 257), (2304, 768, 1030), (19200, 1024, 200)])
def test_mmq_persistent_pairs(rows, cols, m):
    """More pair tiles than co-resident CTA pairs: every pair walks several tiles; the final partial
    round is split along K into workspace partials (8192 x 1024 x 640: 96 tiles; 19200 x 1024: 75
    tiles = one full round + 1 tile split 2 ways); ragged token tails take the plain-store path
    (m = 257: rows not 16-byte aligned, so no bulk row stores at all)."""
    rng = np.random.default_rng(rows + m)
    w = rng.standard_normal((rows, cols)) * 0.05
    q = P.quantize_tensor(torch.from_numpy(w.astype(np.float32)).cuda())
    X = rng.standard_normal((cols, m)).astype(np.float32)
    Y = P.fused_matmul(q, torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
    exact, bound = mmq_bound(q.payload().cpu().numpy(), rows, cols, X)
    assert np.all(np.abs(Y - exact) <= bound), np.max(np.abs(Y - exact) / bound)


def test_mmq_bf16_output_matches_fp32():
    rng = np.random.default_rng(9)
    q = P.quantize_tensor(torch.from_numpy((rng.standard_normal((1536, 1024)) * 0.05).astype(np.float32)).cuda())
    X = torch.from_numpy(rng.standard_normal((1024, 384)).astype(np.float32)).cuda()
    y32 = P.compute._matmul_device(q, X, torch.float32, P.compute.perf_limbs(384))
    y16 = P.compute._matmul_device(q, X, torch.bfloat16, P.compute.perf_limbs(384))
    assert y16.dtype == torch.bfloat16
    torch.testing.assert_close(y16, y32.to(torch.bfloat16), rtol=0, atol=0)


@pytest.mark.parametrize("m", [16, 64, 200])
@pytest.mark.parametrize("bad", [float("nan"), float("inf")])
def test_mmq_nonfinite_input_raises(m, bad):
    """The batched paths check X for non-finite values inside their activation rotation (no separate
    pass): same DomainError as the reference, and the device flag is left clear for the next call."""
    rng = np.random.default_rng(m)
    q = P.quantize_tensor(rng.standard_normal((256, 512)) * 0.1)
    X = torch.from_numpy(rng.standard_normal((512, m)).astype(np.float32)).cuda()
    X[300, m - 1] = bad
    with pytest.raises(P.DomainError, match="non-finite"):
        P.fused_matmul(q, X)
    X[300, m - 1] = 0.0
    Y = P.fused_matmul(q, X)  # clean call afterwards
    assert torch.isfinite(Y).all()


@pytest.mark.parametrize("rows,cols,m", [(300, 512, 16), (1000, 768, 64), (4352, 1024, 300), (640, 256, 2048)])
@pytest.mark.parametrize("asym", [False, True])
def test_mmq_sub_scales(rows, cols, m, asym):
    """Variant ss (per-32 sub-scales, 116-byte blocks) on K5: A = d_m t with the sub-block's scale."""
    rng = np.random.default_rng(rows + m)
    w = rng.standard_normal((rows, cols)) * np.repeat(rng.uniform(0.01, 0.3, (1, cols // 32)), 32, axis=1)
    q = P.quantize_tensor(w, P.QuantConfig(variant="ss", symmetric=not asym))
    assert q.mmq_ok() and not q.fast_layout()
    X = rng.standard_normal((cols, m)).astype(np.float32)
    Y = P.fused_matmul(q, torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
    exact, bound = mmq_bound(q.payload().cpu().numpy(), rows, cols, X, ss=True)
    assert np.all(np.abs(Y - exact) <= bound), np.max(np.abs(Y - exact) / bound)


@pytest.mark.parametrize("n", [32, 64, 128, 512])
@pytest.mark.parametrize("rows,cols,m", [(300, 512, 16), (1000, 1536, 100), (640, 1024, 2048)])
@pytest.mark.parametrize("asym", [False, True])
def test_mmq_block_sizes(n, rows, cols, m, asym):
    """block_n 32..128 on K5: per-32 scale/zero-point tables (several blocks per 128-k stage) and the
    n-point activation rotation x'' = H_n x / sqrt(n)."""
    rng = np.random.default_rng(n + rows + m)
    w = rng.standard_normal((rows, cols)) * 0.05 + (0.02 if asym else 0.0)
    q = P.quantize_tensor(w, P.QuantConfig(block_n=n, symmetric=not asym))
    assert q.mmq_ok()
    X = rng.standard_normal((cols, m)).astype(np.float32)
    Y = P.fused_matmul(q, torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
    exact, bound = mmq_bound(q.payload().cpu().numpy(), rows, cols, X, n=n)
    assert np.all(np.abs(Y - exact) <= bound), np.max(np.abs(Y - exact) / bound)


@pytest.mark.parametrize("asym", [False, True])
def test_mmq_sub_scales_512(asym):
    """Variant ss at block_n 512: 64-wide sub-blocks, so both 32-k groups of a sub-block share its scale."""
    rng = np.random.default_rng(51)
    rows, cols, m = 700, 1536, 200
    w = rng.standard_normal((rows, cols)) * np.repeat(rng.uniform(0.01, 0.3, (1, cols // 64)), 64, axis=1)
    q = P.quantize_tensor(w, P.QuantConfig(block_n=512, variant="ss", symmetric=not asym))
    assert q.mmq_ok()
    X = rng.standard_normal((cols, m)).astype(np.float32)
    Y = P.fused_matmul(q, torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
    exact, bound = mmq_bound(q.payload().cpu().numpy(), rows, cols, X, ss=True, n=512)
    assert np.all(np.abs(Y - exact) <= bound), np.max(np.abs(Y - exact) / bound)


@pytest.mark.parametrize("variant", ["s", "ss"])
def test_mmq_huge_scale_takes_exact_path(variant):
    """A block whose scale is >= 2^15 would overflow K5's binary16 A = d t; such tensors take a path
    with fp32 scales instead (the K4 GEMV for the default format, the exact generic kernel otherwise),
    so fused_matmul stays finite and within the perf-mode bound."""
    rng = np.random.default_rng(77)
    w = rng.standard_normal((256, 512)) * 0.05
    w[3, :256] *= 2.0e6  # sigma ~1e5 -> stored scale saturates near 65504
    q = P.quantize_tensor(w, P.QuantConfig(variant=variant))
    assert not q.k5_range_ok()
    X = rng.standard_normal((512, 100)).astype(np.float32)  # k > 64: the K5 range
    Y = P.fused_matmul(q, torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
    exact, bound = mmq_bound(q.payload().cpu().numpy(), 256, 512, X, ss=variant == "ss")
    assert np.all(np.isfinite(Y))
    assert np.all(np.abs(Y - exact) <= bound), np.max(np.abs(Y - exact) / bound)


@pytest.mark.parametrize("fmt", [dict(variant="ss"), dict(block_n=64), dict(block_n=512, variant="ss"),
                                 dict(block_n=128, symmetric=False)])
@pytest.mark.parametrize("m", [1, 3, 7])
def test_small_k_other_formats_on_k5(fmt, m):
    """Variant ss / block_n != 256 at k < 8 (incl. the k = 1 GEMV): K5 on X zero-padded to 8 tokens,
    within the K5 bound per column; the padded columns never leak into the result's shape."""
    rng = np.random.default_rng(m + len(str(fmt)))
    rows, cols = 700, 1536
    w = rng.standard_normal((rows, cols)) * np.repeat(rng.uniform(0.01, 0.3, (1, cols // 32)), 32, axis=1)
    q = P.quantize_tensor(w, P.QuantConfig(**fmt))
    assert q.mmq_ok() and not q.fast_layout()
    X = rng.standard_normal((cols, m)).astype(np.float32)
    Y = P.fused_matmul(q, torch.from_numpy(X).cuda())
    assert tuple(Y.shape) == (rows, m)
    exact, bound = mmq_bound(q.payload().cpu().numpy(), rows, cols, X, ss=fmt.get("variant") == "ss",
                             n=fmt.get("block_n", 256))
    Yn = Y.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(Yn - exact) <= bound), np.max(np.abs(Yn - exact) / bound)
    if m == 1:  # fused_matvec goes the same way
        y = P.fused_matvec(q, torch.from_numpy(X[:, 0]).cuda()).cpu().numpy().astype(np.float64).reshape(-1)
        assert np.all(np.abs(y - exact[:, 0]) <= bound[:, 0])
