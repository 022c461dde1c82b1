"""GPU parity at the shapes the benchmarks time (VERDICT r01 "parity-test the configs you benchmark").

* C3 (BASELINE configs[2]): full Llama-3-8B-shaped layers (14336x4096, 4096x14336, 4096x4096,
  1024x4096) quantized on the GPU, multiplied by fused_matmul at M = 16 / 32 / 64 (K5b, tcgen05
  kind::i8) and M = 128 / 1024 / 2048 (K5, tcgen05 kind::f16 CTA pairs; 14336x4096 at M = 1024 is the
  split-K tail round).  256 sampled rows (first and last included) are checked against the oracle's
  exact fp64 product of the decoded weights with the a-priori bound of the path:
    K5  : test_gpu_mmq.mmq_bound   (f16 rotated activations, exact f16 A = d t);
    K5b : chain_bound at L = 2     (16-bit fixed-point activations per (token, block)).
* Reference pins: the LAST rows of the full layer are replaced by the reference's C3 row samples
  (tests/golden/make_golden.py C3_EXTRA, produced by running the reference's fused_matmul), so the
  reference's own outputs are compared with the kernel running at the full shape.
* C5 (configs[4]): a chain stage with K = 28672 (7 K-chunk partials per output).
* C4 (configs[3]): the decoder stack at Llama-3-8B width (RMSNorm-in-chain with the whole 4096-wide
  input in one CTA, 16 blocks).
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import itq3_oracle as O
from test_gpu_mmq import mmq_bound

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2603_27914_b200")

HERE = os.path.join(os.path.dirname(__file__), "golden")
H256 = O.hadamard(256)
C3_SHAPES = [(14336, 4096), (4096, 14336), (4096, 4096), (1024, 4096)]


def chain_bound_cols(payload, rows, cols, X, limbs):
    """test_gpu_stack.chain_bound for every column of X at once: (exact, bound), each rows x m."""
    n, nb = 256, cols // 256
    X = np.asarray(X, np.float64)
    deq = O.dequantize(payload, rows, cols, n, False)
    quants, sb, zb, _ = O.split_payload(payload, n, False)
    codes, _ = O.unpack_planes(quants, n)
    t = codes.astype(np.float64) - np.trunc(O.f16_value(zb))[:, None]
    t1 = np.maximum(np.abs(t).sum(axis=1), codes.astype(np.float64).sum(axis=1)).reshape(rows, nb)  # see chain_bound
    ht1 = np.abs(t @ H256).sum(axis=1).reshape(rows, nb)
    d = O.f16_value(sb).reshape(rows, nb)
    xb = X.T.reshape(-1, nb, n)                                         # (m, nb, n)
    mx = np.abs(xb).max(axis=2)
    e_in = np.where(mx > 0, np.floor(np.log2(np.where(mx > 0, mx, 1.0))) - 21, 0)
    xi = np.rint(xb * 2.0 ** -e_in[:, :, None])
    amax = np.abs(xi @ H256).max(axis=2)
    bl = np.where(amax > 0, np.floor(np.log2(np.where(amax > 0, amax, 1.0))) + 1, 0)
    k = np.maximum(0, bl - (8 * limbs - 2))
    bound = (d * t1 / 32.0) @ (2.0 ** (e_in + k)).T + (d * ht1 / 32.0) @ (2.0 ** e_in).T
    return deq @ X, bound + 1e-5 * (np.abs(deq) @ np.abs(X))


def sample_rows(rows, n=256, seed=0):
    rng = np.random.default_rng(seed + rows)
    r = rng.choice(np.arange(1, rows - 1), size=min(n, rows) - 2, replace=False)
    return np.unique(np.concatenate([[0, rows - 1], r]))


def row_payload(q, rows_idx):
    nbytes = q.cols // 256 * 100
    pay = q.payload().view(q.rows, nbytes)
    return pay[torch.as_tensor(rows_idx, device=pay.device)].cpu().numpy().reshape(-1)


def layer(rows, cols, seed, embed=None):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    w = torch.randn((rows, cols), generator=g, device="cuda").mul_(cols ** -0.5)
    if embed is not None:
        w[rows - embed.shape[0]:] = torch.from_numpy(embed).cuda()
    return P.quantize_tensor(w)


def check(q, X, Y, rows_idx):
    pay = row_payload(q, rows_idx)
    Xn = X.cpu().numpy().astype(np.float64)
    Yn = Y.cpu().numpy().astype(np.float64)[rows_idx]
    m = X.shape[1]
    if P.compute.MMQ_MIN_TOKENS <= m <= P.compute.MMQ8_MAX_TOKENS:
        exact, bound = chain_bound_cols(pay, len(rows_idx), q.cols, Xn, limbs=2)
    else:
        exact, bound = mmq_bound(pay, len(rows_idx), q.cols, Xn)
    err = np.abs(Yn - exact)
    assert np.all(err <= bound), float(np.max(err / bound))
    return exact, bound


@pytest.mark.parametrize("rows,cols", C3_SHAPES)
@pytest.mark.parametrize("m", [16, 32, 64, 128, 1024, 2048])
def test_c3_full_shape(rows, cols, m):
    q = layer(rows, cols, seed=rows + cols)
    g = torch.Generator(device="cuda")
    g.manual_seed(m)
    X = torch.randn((cols, m), generator=g, device="cuda")
    Y = P.fused_matmul(q, X)
    assert Y.shape == (rows, m) and bool(torch.isfinite(Y).all())
    check(q, X, Y, sample_rows(rows))


def _c3_golden():
    with open(os.path.join(HERE, "full_digests.json")) as f:
        return json.load(f)["c3"][1:]


@pytest.mark.parametrize("case", _c3_golden(), ids=lambda c: f"{c['rows']}x{c['cols']}_m{c['m']}")
def test_c3_reference_rows_at_full_shape(case):
    """The reference's fused_matmul output for a row sample, embedded as the last rows of a full
    Llama-3-8B-shaped layer (14336 x 4096 or 4096 x 14336)."""
    r, cols, m = case["rows"], case["cols"], case["m"]
    rows = 14336 if cols == 4096 else 4096
    w = O.generate_weights("gaussian", r, cols, seed=case["seed"]).astype(np.float32)
    X = np.random.default_rng(case["x_seed"]).standard_normal((cols, m)).astype(np.float32)
    q = layer(rows, cols, seed=7 * rows + m, embed=w)
    idx = np.arange(rows - r, rows)
    pay = row_payload(q, idx)
    ref_pay, _ = O.quantize_payload(w)
    assert np.array_equal(pay, ref_pay.reshape(-1)), "row-shard encode differs from the reference sample's container"
    Y = P.fused_matmul(q, torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)[idx]
    Y_ref = np.load(os.path.join(HERE, case["y_file"]))
    if P.compute.MMQ_MIN_TOKENS <= m <= P.compute.MMQ8_MAX_TOKENS:
        _, bound = chain_bound_cols(pay, r, cols, X, limbs=2)
    else:
        _, bound = mmq_bound(pay, r, cols, X)
    err = np.abs(Y - Y_ref)
    assert np.all(err <= bound), float(np.max(err / bound))


def test_chain_c5_k28672():
    """C5's down projection width: K = 28672 -> 112 blocks -> 7 K-chunk partials per output, folded
    in fixed order by the next stage's loads and the final fold."""
    from test_gpu_stack import build, chain_bound, lo_flags

    from paper_2603_27914_b200.stack import LinearStack

    shapes = [(28672, 512), (1024, 28672), (512, 1024)]
    qs = build(41, shapes=shapes)
    st = LinearStack(qs, limbs=3, mode="chain")
    x = np.random.default_rng(5).standard_normal(512).astype(np.float32)
    out = st.forward(x).copy()  # forward returns the stack's reused output buffer
    xin = x.astype(np.float64)
    for i, q in enumerate(qs):
        y = st.stage_output(i).cpu().numpy().astype(np.float64)
        exact, bound = chain_bound(q.payload().cpu().numpy(), q.rows, q.cols, xin, 3, **lo_flags(st, i))
        assert np.all(np.abs(y - exact) <= bound), (i, float(np.max(np.abs(y - exact) / bound)))
        if i + 1 < len(qs):
            xin = y[: qs[i + 1].cols]
    np.testing.assert_array_equal(out, st.stage_output(len(qs) - 1).cpu().numpy())
    for _ in range(2):  # replays reproduce bit for bit
        np.testing.assert_array_equal(st.forward(x), out)


def test_decoder_llama3_8b_width():
    """DecoderStack at Llama-3-8B width (hidden 4096, ffn 14336, 32 / 8 heads), 2 layers, vs the
    plain torch fp32 step with the dequantised weights (tolerance as tests/test_gpu_decoder.py)."""
    from paper_2603_27914_b200.decoder import DecoderStack

    dev = torch.device("cuda", 0)
    st = DecoderStack(layers=2, max_ctx=128, seed=11, dev=dev, serving=False, shapes=dict(vocab=16384))
    g = torch.Generator(device=dev)
    g.manual_seed(12)
    k_hist, v_hist = [[] for _ in range(2)], [[] for _ in range(2)]
    for pos in range(40):
        x = torch.randn(4096, generator=g, device=dev)
        got = st.step(x).clone()
        want = st.reference_step(x, pos, k_hist, v_hist)
        err = float((got - want).norm() / want.norm())
        assert err < 1e-4, (pos, err)
        lerr = float((st.logits - st.ref_logits).norm() / st.ref_logits.norm())
        assert lerr < 1e-4, (pos, lerr)
