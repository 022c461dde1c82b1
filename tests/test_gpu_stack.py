"""GPU: the decode-chain harness (stack.py) in both modes -- the persistent chain kernel
(csrc/chain.cu) and the per-stage kernels -- against the CPU oracle, stage by stage.

Each stage's output is checked against the exact fp64 product of the oracle-decoded weights
with the GPU's own previous-stage output (so errors do not compound), within the perf-mode
bound of test_gpu_parity.perf_bound (24-bit rotated activations, fp32 accumulation)."""

import numpy as np
import pytest
import torch

from oracle import itq3_oracle as O

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2603_27914_b200")
from paper_2603_27914_b200.stack import LinearStack  # noqa: E402

H256 = O.hadamard(256)


def chain_bound(payload, rows, cols, x, limbs=3, lo_in=False, lo_x0=False, lo_out=False, nch=1):
    """A-priori error bound of the chain kernel's stage output vs the exact fp64 product.

    The chain rotates in integers: x -> x_int = rint(x / s_in), s_in = 2^(ilogb(max|x_b|) - 21),
    exact butterfly, x' rounded to |q| <= 2^(8L-2) by a shift k (csrc/chain.cu).  Per block:
        |err| <= d/16 * ( max(|t|_1, |c|_1) * 2^(e_in+k) / 2 + |H t|_1 * s_in / 2 )
    (|c|_1: the chain subtracts the exact sum of x'; |t|_1: K3 / K5b subtract the rounded sum)
    plus 1e-5 * sum |w_hat| |x| for fp32 accumulation (also covers the K3 path of mode="kernels").

    The symmetric single-GPU chain kernel (LO) takes its input as y = H_16 x per 16-element group
    (lo_in): s_in comes from max|y|, the rounding happens on y, so the rounding term weighs |H_hi t|_1
    (H_16 over the group index only); its zero-point correction converts a 16-term integer sum to fp32
    (|v0| 2^-24 s_in d |z|).  lo_x0: y was formed in-kernel from x in fp32 (4 adds: 4u sum_group |x|).
    lo_out: the stored output is H_16 y of fp32 sums over nch K-chunk partials, read back through H_16^-1
    in fp64: (6 + nch) u sum_{16-row group} |w_hat| |x| more (two radix-4 rounds of 3 roundings each).
    """
    n = 256
    nb = cols // n
    deq = O.dequantize(payload, rows, cols, n, False)
    quants, sb, zb, _ = O.split_payload(payload, n, False)
    codes, _ = O.unpack_planes(quants, n)
    z = np.trunc(O.f16_value(zb))
    t = codes.astype(np.float64) - z[:, None]
    # the chain kernel corrects with the exact sum of x' (256 x_0): its limb-rounding term is |c|_1;
    # K3/K5b correct with the rounded sum: |t|_1 -- the max covers both
    t1 = np.maximum(np.abs(t).sum(axis=1), codes.astype(np.float64).sum(axis=1)).reshape(rows, nb)
    d = O.f16_value(sb).reshape(rows, nb)
    xb = np.asarray(x, np.float64).reshape(nb, n)
    mag = np.abs(deq) @ np.abs(np.asarray(x, np.float64))
    if not lo_in:
        ht1 = np.abs(t @ H256).sum(axis=1).reshape(rows, nb)
        mx = np.abs(xb).max(axis=1)
        e_in = np.where(mx > 0, np.floor(np.log2(np.where(mx > 0, mx, 1.0))) - 21, 0)
        xi = np.rint(xb * 2.0 ** -e_in[:, None])
        amax = np.abs(xi @ H256).max(axis=1)
        extra = 0.0
    else:
        H16 = O.hadamard(16)
        yb = xb.reshape(nb, 16, 16) @ H16  # [block, group a, b]: H_16 over b
        th = np.abs(np.einsum("ac,rcb->rab", H16, t.reshape(-1, 16, 16))).sum(axis=2)  # |H_hi t| per group a
        ht1 = th.sum(axis=1).reshape(rows, nb)
        mx = np.abs(yb).reshape(nb, -1).max(axis=1)
        e_in = np.where(mx > 0, np.floor(np.log2(np.where(mx > 0, mx, 1.0))) - 21, 0)
        yi = np.rint(yb * 2.0 ** -e_in[:, None, None])
        amax = np.abs(np.einsum("ac,ncb->nab", H16, yi)).reshape(nb, -1).max(axis=1)
        v0 = np.abs(yi[:, 0, :].sum(axis=1))
        extra = d * np.abs(z).reshape(rows, nb) * (v0 * 2.0 ** (e_in - 24))[None, :]
        if lo_x0:
            dx = 4 * 2.0 ** -24 * np.abs(xb).reshape(nb, 16, 16).sum(axis=2)  # [block, a]
            extra = extra + d / 16.0 * np.einsum("rna,na->rn", th.reshape(rows, nb, 16), dx)
    bl = np.where(amax > 0, np.floor(np.log2(np.where(amax > 0, amax, 1.0))) + 1, 0)
    k = np.maximum(0, bl - (8 * limbs - 2))
    bound = (d / 16.0 * (t1 * 2.0 ** (e_in + k)[None, :] / 2 + ht1 * 2.0 ** e_in[None, :] / 2) + extra).sum(axis=1)
    bound = bound + 1e-5 * mag
    if lo_out:
        full = rows // 16 * 16
        gm = np.repeat(mag[:full].reshape(-1, 16).sum(axis=1), 16)
        bound[:full] += (6 + nch) * 2.0 ** -24 * gm
    return deq @ np.asarray(x, np.float64), bound


def lo_flags(st, i):
    """chain_bound's LO arguments for stage i of a LinearStack run (see LinearStack.lo)."""
    lo = st.mode == "chain" and st.sym and st.lo_kernel
    return dict(lo_in=lo, lo_x0=lo and (i == 0 or st.independent), lo_out=bool(lo and st.lo[i]),
                nch=int(st.nch[i]) if lo else 1)


SHAPES = [(26112, 256), (768, 512), (512, 512), (1280, 512), (512, 1024), (4608, 512), (256, 4608), (9000, 256), (400, 8960),
          (8960, 256), (300, 8704)]


def build(seed, shapes=SHAPES, asym=False):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    qs = []
    for r, c in shapes:
        w = torch.randn((r, c), generator=g, device="cuda") / np.sqrt(c)
        qs.append(P.quantize_tensor(w, P.QuantConfig(symmetric=not asym)))
    return qs


@pytest.mark.parametrize("mode", ["chain", "kernels"])
@pytest.mark.parametrize("asym", [False, True])
def test_stack_matches_oracle_stagewise(mode, asym):
    qs = build(5, asym=asym)
    pays = [q.payload().cpu().numpy() for q in qs]
    st = LinearStack(qs, limbs=3, mode=mode)
    x = np.random.default_rng(0).standard_normal(qs[0].cols).astype(np.float32)
    out = st.forward(x).copy()
    xin = x.astype(np.float64)
    for i, q in enumerate(qs):
        y = st.stage_output(i).cpu().numpy().astype(np.float64)
        exact, bound = chain_bound(pays[i], q.rows, q.cols, xin, 3, **lo_flags(st, i))
        assert np.all(np.abs(y - exact) <= bound), (mode, i, np.max(np.abs(y - exact) / bound))
        if i + 1 < len(qs):
            xin = st.stage_output(i).cpu().numpy().astype(np.float64)[: qs[i + 1].cols]
    np.testing.assert_array_equal(out, st.stage_output(len(qs) - 1).cpu().numpy())


def test_chain_replay_deterministic_and_matches_kernels():
    qs = build(9)
    a = LinearStack(qs, mode="chain")
    b = LinearStack(qs, mode="kernels")
    x = np.random.default_rng(1).standard_normal(qs[0].cols).astype(np.float32)
    ya = a.forward(x).copy()
    for _ in range(3):
        np.testing.assert_array_equal(a.forward(x), ya)  # graph replays are bitwise reproducible
    yb = b.forward(x)
    np.testing.assert_allclose(ya, yb, rtol=1e-3, atol=1e-4 * np.abs(yb).max())


def test_chain_beyond_smem_descriptor_cache():
    """170 stages: descriptors past the kernel's shared-memory cache (136) come from global memory
    with the work split computed per stage; every stage still matches the oracle bound."""
    shapes = [(512, 256), (256, 512)] * 85
    qs = build(21, shapes=shapes)
    pays = [q.payload().cpu().numpy() for q in qs]
    st = LinearStack(qs, limbs=3, mode="chain")
    x = np.random.default_rng(3).standard_normal(qs[0].cols).astype(np.float32)
    out = st.forward(x).copy()
    xin = x.astype(np.float64)
    for i, q in enumerate(qs):
        y = st.stage_output(i).cpu().numpy().astype(np.float64)
        if i >= 140 or i % 20 == 0:
            exact, bound = chain_bound(pays[i], q.rows, q.cols, xin, 3, **lo_flags(st, i))
            assert np.all(np.abs(y - exact) <= bound), (i, np.max(np.abs(y - exact) / bound))
        if i + 1 < len(qs):
            xin = y[: qs[i + 1].cols]
    np.testing.assert_array_equal(out, st.stage_output(len(qs) - 1).cpu().numpy())
