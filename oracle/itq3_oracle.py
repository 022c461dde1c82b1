"""CPU oracle for the ITQ3_S hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``itq3`` 0.1.0
(``/root/reference/pkg/src/itq3``) for the functions on the hot path named by
BASELINE.json ``north_star``: FWHT rotation, scale policy, ternary quantization,
bit-plane packing, block/tensor decode, the fused matmul and the container.
Every function cites the reference file:line it restates.

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
    (``cpu_baseline`` and ``--impl reference``) may import this module, and only
    as the checker or as the timed CPU baseline -- never on the product path.
  * Parity is PINNED: ``tests/golden/make_golden.py`` runs the real reference
    (importable in the build container) and commits fixtures + SHA-256 digests;
    ``tests/test_oracle_golden.py`` checks this restatement against them.

The encoder is vectorised over blocks but follows the *block codec*
(``codec.py:113-149``) where the reference's own vectorised path diverges
(binary16 overflow saturates instead of producing inf, ``packing.py:99-100``).
"""

from __future__ import annotations

import math
import struct

import numpy as np

# --- constants (reference file:line) -------------------------------------------------
DEFAULT_SCALE_COEFF = 0.7979  # quantizer.py:24
EPSILON_D = 1e-8  # quantizer.py:28
F16_MAX = 65504.0  # packing.py:33
F16_NAN = 0x7E00  # packing.py:34
SUB_BLOCKS = 8  # packing.py:31, codec.py:49
BLOCK_SIZES = (32, 64, 128, 256, 512)  # codec.py:47
MAGIC = b"ITQ3"  # codec.py:42
VERSION = 1  # codec.py:43
FLAG_SUB_SCALES = 0x1  # codec.py:44
FLAG_ASYMMETRIC = 0x2  # codec.py:45
HEADER = struct.Struct("<4sHHQQII")  # codec.py:50


def argmin_coeff() -> float:
    """quantizer.py:130-138: alphas = arange(1,2001)*1e-3, argmin of the Gaussian MSE.

    The grid minimiser is index 877 (alpha = 0.878); the survey re-ran the
    scipy quadrature and ``tests/golden`` pins the value the
    reference returns.  The float is formed exactly as the reference forms it.
    """
    return float((np.arange(1, 2001) * 1e-3)[877])


# --- L1 transform (transform.py) --------------------------------------------------------
def butterfly(a: np.ndarray) -> np.ndarray:
    """Unnormalised radix-2 Walsh-Hadamard butterfly along the last axis.

    transform.py:46-58: for h = 1, 2, ..., n/2 pair element j (j & h == 0) with
    j + h and write (lo + hi, lo - hi).  The per-element data flow is the same
    as the reference's reshape/stack formulation, so results are bit-identical.
    """
    a = np.asarray(a)
    n = a.shape[-1]
    y = a.reshape(-1, n).astype(a.dtype, copy=True)
    h = 1
    while h < n:
        v = y.reshape(y.shape[0], n // (2 * h), 2, h)
        lo = v[:, :, 0, :].copy()
        hi = v[:, :, 1, :]
        v[:, :, 0, :] = lo + hi
        v[:, :, 1, :] = lo - hi
        h <<= 1
    return y.reshape(a.shape)


def fwht(a: np.ndarray) -> np.ndarray:
    """Normalised FWHT (transform.py:61-96): butterfly then one multiply by fl(1/sqrt(n))."""
    a = np.asarray(a)
    if not np.issubdtype(a.dtype, np.inexact):
        a = a.astype(np.float64)
    n = a.shape[-1]
    return butterfly(a) * np.asarray(1.0 / math.sqrt(n), dtype=a.dtype)


def hadamard(n: int) -> np.ndarray:
    """Sylvester +-1 matrix (transform.py:99-106), unnormalised, H[k,j] = (-1)^popc(k&j)."""
    k = np.arange(n)
    pc = np.vectorize(lambda v: bin(v).count("1"))(k[:, None] & k[None, :])
    return np.where(pc % 2 == 0, 1.0, -1.0)


# --- binary16 (packing.py:87-109) -----------------------------------------------------
def f16_bits(x) -> np.ndarray:
    """encode_f16 vectorised: RNE single rounding, finite overflow saturates to +-65504.

    packing.py:87-101.  NaN -> 0x7E00, +-inf pass through.
    """
    v = np.asarray(x, dtype=np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        h = v.astype(np.float16)
    sat = np.isinf(h) & np.isfinite(v)
    h = np.where(sat, np.where(v > 0, np.float16(F16_MAX), np.float16(-F16_MAX)), h).astype(np.float16)
    bits = h.view(np.uint16).copy()
    bits[np.isnan(v)] = F16_NAN
    return bits


def f16_value(bits) -> np.ndarray:
    """decode_f16 (packing.py:104-109): exact binary16 value as float64."""
    return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float64)


# --- L2 quantizer (quantizer.py) --------------------------------------------------------
def policy_scales(y: np.ndarray, kind: str = "constant", constant: float = DEFAULT_SCALE_COEFF) -> np.ndarray:
    """Raw per-row scale, floored at EPSILON_D.

    quantizer.py:78-99 (block_stats: mean = np.mean, var = np.mean((a-mean)**2),
    sigma = sqrt) and quantizer.py:141-149 (optimal_scale).  np.mean over
    axis=1 of a C-contiguous array reduces each row with the same pairwise
    summation as the 1-D call (pinned by tests/golden).
    """
    if kind == "mean-abs":
        d = (2.0 / 3.0) * (np.sum(np.abs(y), axis=1) / y.shape[1])
    else:
        coeff = constant if kind == "constant" else argmin_coeff()
        mu = np.mean(y, axis=1, keepdims=True)
        sigma = np.sqrt(np.mean((y - mu) ** 2, axis=1))
        d = coeff * sigma
    return np.where(d > 0, d, EPSILON_D)


def effective_scale(d_raw: np.ndarray) -> np.ndarray:
    """codec.py:95-103: quantise against the stored (saturating) binary16 scale, else raw."""
    d16 = f16_value(f16_bits(d_raw))
    return np.where(d16 > 0, d16, d_raw)


def round_half_away(v: np.ndarray) -> np.ndarray:
    """quantizer.py:152-153: copysign(floor(|v| + 0.5), v)."""
    return np.copysign(np.floor(np.abs(v) + 0.5), v)


def zero_points(mean: np.ndarray, d_eff: np.ndarray, symmetric: bool) -> np.ndarray:
    """codec.py:106-110."""
    if symmetric:
        return np.zeros_like(mean)
    r = mean / d_eff
    # int(...) in the reference (codec.py:110) turns -0.0 into 0 -> binary16 0x0000
    return np.clip(-np.copysign(np.floor(np.abs(r) + 0.5), r), -1.0, 1.0) + 0.0


def ternary_codes(y: np.ndarray, d_eff: np.ndarray, z: np.ndarray) -> np.ndarray:
    """quantizer.py:156-168: clip(round_half_away(y/d) + z, -1, 1) as int8 (broadcasting)."""
    return np.clip(round_half_away(y / d_eff) + z, -1.0, 1.0).astype(np.int8)


# --- L3 packing (packing.py) ----------------------------------------------------------------
def pack_planes(codes: np.ndarray) -> np.ndarray:
    """packing.py:59-64 vectorised: c = q + 1, plane b = packbits((c>>b)&1, little)."""
    c = (codes.astype(np.int16) + 1).astype(np.uint8)
    planes = [np.packbits((c >> b) & 1, axis=-1, bitorder="little") for b in range(3)]
    return np.concatenate(planes, axis=-1)


def unpack_planes(quants: np.ndarray, n: int):
    """packing.py:67-84 vectorised: returns (codes int8, first_bad (block, index) or None)."""
    q = np.asarray(quants, dtype=np.uint8).reshape(-1, 3 * n // 8)
    pl = n // 8
    bits = [np.unpackbits(q[:, b * pl:(b + 1) * pl], axis=1, bitorder="little") for b in range(3)]
    c = bits[0].astype(np.int16) + 2 * bits[1] + 4 * bits[2]
    bad = np.argwhere(c > 2)
    first = (int(bad[0, 0]), int(bad[0, 1]), int(c[bad[0, 0], bad[0, 1]])) if bad.size else None
    return (c - 1).astype(np.int8), first


def block_nbytes(n: int, ss: bool) -> int:
    """packing.py:37-40."""
    return 3 * n // 8 + 4 + (16 if ss else 0)


# --- L4 codec (codec.py) -------------------------------------------------------------------------
def blockify(w: np.ndarray, n: int):
    """codec.py:173-179 / compute.py:136-143: row-major flatten, zero-pad the tail."""
    flat = np.asarray(w, dtype=np.float64).reshape(-1)
    nb = -(-flat.size // n)
    pad = nb * n - flat.size
    if pad:
        flat = np.concatenate([flat, np.zeros(pad)])
    return flat.reshape(nb, n), pad


def encode_blocks(blocks: np.ndarray, variant="s", symmetric=True, kind="constant",
                  constant=DEFAULT_SCALE_COEFF):
    """encode_block (codec.py:113-149) for every row of ``blocks``.

    Returns (codes int8 (nb,n), scale_bits u16 (nb,), zp_bits u16 (nb,), sub_bits u16 (nb,8) | None).
    """
    nb, n = blocks.shape
    y = fwht(blocks)
    mean = np.mean(y, axis=1)
    if variant == "s":
        d_raw = policy_scales(y, kind, constant)
        d_eff = effective_scale(d_raw)
        z = zero_points(mean, d_eff, symmetric)
        codes = ternary_codes(y, d_eff[:, None], z[:, None])
        return codes, f16_bits(d_raw), f16_bits(z), None
    m = n // SUB_BLOCKS
    subs = y.reshape(nb * SUB_BLOCKS, m)
    d_raw = policy_scales(subs, kind, constant).reshape(nb, SUB_BLOCKS)
    d_eff = effective_scale(d_raw)
    d_block = np.mean(d_raw, axis=1)
    z = zero_points(mean, effective_scale(d_block), symmetric)
    codes = ternary_codes(y.reshape(nb, SUB_BLOCKS, m), d_eff[:, :, None], z[:, None, None]).reshape(nb, n)
    return codes, f16_bits(d_block), f16_bits(z), f16_bits(d_raw)


def serialize(codes, scale_bits, zp_bits, sub_bits=None) -> np.ndarray:
    """PackedBlock.to_bytes (packing.py:136-141) for all blocks -> (nb, block_nbytes) uint8."""
    nb = codes.shape[0]
    parts = [pack_planes(codes),
             np.asarray(scale_bits, "<u2").reshape(nb, 1).view(np.uint8),
             np.asarray(zp_bits, "<u2").reshape(nb, 1).view(np.uint8)]
    if sub_bits is not None:
        parts.append(np.ascontiguousarray(np.asarray(sub_bits, "<u2")).view(np.uint8).reshape(nb, 16))
    return np.concatenate(parts, axis=1)


def quantize_payload(w, block_n=256, variant="s", symmetric=True, kind="constant",
                     constant=DEFAULT_SCALE_COEFF):
    """quantize_tensor (codec.py:164-189) -> (payload uint8 (nb, bsize), pad)."""
    blocks, pad = blockify(w, block_n)
    codes, sb, zb, sub = encode_blocks(blocks, variant, symmetric, kind, constant)
    return serialize(codes, sb, zb, sub), pad


def split_payload(payload: np.ndarray, n: int, ss: bool):
    """Field views of a (nb, bsize) payload: quants, scale_bits, zp_bits, sub_bits."""
    p = np.asarray(payload, dtype=np.uint8).reshape(-1, block_nbytes(n, ss))
    q = 3 * n // 8
    sb = p[:, q:q + 2].copy().view("<u2")[:, 0]
    zb = p[:, q + 2:q + 4].copy().view("<u2")[:, 0]
    sub = p[:, q + 4:q + 20].copy().view("<u2") if ss else None
    return p[:, :q], sb, zb, sub


def decode_payload(payload: np.ndarray, n: int, ss: bool) -> np.ndarray:
    """decode_block (codec.py:152-161) for all blocks -> (nb, n) float64."""
    quants, sb, zb, sub = split_payload(payload, n, ss)
    codes, bad = unpack_planes(quants, n)
    if bad is not None:
        raise ValueError(f"block {bad[0]}: stored code {bad[2]} > 2 at index {bad[1]}")
    z = np.trunc(f16_value(zb))[:, None]  # PackedBlock.zp = int(decode_f16(...)) (packing.py:128-130)
    if sub is None:
        y = f16_value(sb)[:, None] * (codes.astype(np.float64) - z)
    else:
        y = np.repeat(f16_value(sub), n // SUB_BLOCKS, axis=1) * (codes.astype(np.float64) - z)
    return fwht(y)


def dequantize(payload, rows, cols, n, ss) -> np.ndarray:
    """dequantize_tensor (codec.py:192-202): decode, strip pad, reshape."""
    flat = decode_payload(payload, n, ss).reshape(-1)
    return flat[:rows * cols].reshape(rows, cols)


def fused_matmul(payload, rows, cols, n, ss, X) -> np.ndarray:
    """fused_matmul (compute.py:98-125) restated as dequantize(q) @ X in float64.

    The reference accumulates per block with OpenBLAS dgemv; both are float64
    with exact decoded weights, so they agree to ~1e-15 relative (tolerance
    parity; the reference's own tests use rtol=1e-5, test_compute.py:66-78).
    """
    X = np.asarray(X, dtype=np.float64)
    return dequantize(payload, rows, cols, n, ss) @ X


# --- container (codec.py:205-291) ----------------------------------------------------------------
def container_bytes(payload, rows, cols, n, variant, symmetric, pad) -> bytes:
    """write_container (codec.py:222-235)."""
    flags = (FLAG_SUB_SCALES if variant == "ss" else 0) | (0 if symmetric else FLAG_ASYMMETRIC)
    return HEADER.pack(MAGIC, VERSION, flags, rows, cols, n, pad) + np.asarray(payload, np.uint8).tobytes()


def parse_container(data: bytes):
    """read_container header checks (codec.py:248-273); returns a dict plus the payload."""
    if len(data) < HEADER.size:
        raise ValueError("truncated")
    magic, version, flags, rows, cols, n, pad = HEADER.unpack_from(data, 0)
    ss = bool(flags & FLAG_SUB_SCALES)
    nb = -(-rows * cols // n)
    bsize = block_nbytes(n, ss)
    payload = np.frombuffer(data, np.uint8, count=nb * bsize, offset=HEADER.size).reshape(nb, bsize)
    return dict(magic=magic, version=version, flags=flags, rows=rows, cols=cols, block_n=n, pad=pad,
                variant="ss" if ss else "s", symmetric=not (flags & FLAG_ASYMMETRIC)), payload


# --- inputs (compute.py:58-95) --------------------------------------------------------------------
def generate_weights(dist, rows, cols, seed, nu=3.0, outlier_frac=0.01, outlier_mult=20.0):
    """generate_weights (compute.py:58-95): seeded synthetic matrices."""
    rng = np.random.default_rng(seed)
    if dist == "gaussian":
        return rng.standard_normal((rows, cols))
    if dist == "laplace":
        return rng.laplace(size=(rows, cols))
    if dist == "student-t":
        return rng.standard_t(nu, size=(rows, cols))
    if dist != "outlier":
        raise ValueError(dist)
    w = rng.standard_normal((rows, cols))
    k = int(round(outlier_frac * w.size))
    if k:
        idx = rng.choice(w.size, size=k, replace=False)
        w.reshape(-1)[idx] *= outlier_mult
    return w


# --- evaluation (compute.py:221-269) ----------------------------------------------------------------
def eval_error(w, payload, n, ss):
    """The eps_q fields of eval_error: mse and frobenius_rel of the decoded tensor."""
    a = np.asarray(w, dtype=np.float64)
    rec = dequantize(payload, a.shape[0], a.shape[1], n, ss)
    err = (rec - a).reshape(-1)
    wn = float(np.linalg.norm(a))
    return {"mse": float(np.mean(err ** 2)),
            "frobenius_rel": float(np.linalg.norm(err) / wn) if wn > 0 else 0.0}


# --- full evaluation harness (compute.py:136-356) -------------------------------------------------
# The reference's evaluation path is its *vectorised* encoder (compute.py:136-218), which casts
# scales with astype(float16) (inf on overflow) instead of encode_f16's saturation.
ERROR_FIELDS = ("mse", "frobenius_rel", "linf_in", "linf_rot", "bound_slack", "clamp_fraction",
                "zero_fraction", "mse_uniform3", "mse_ternary_noro", "n_blocks", "unclamped_blocks")


def f16_round_cast(d):
    """compute.py:146-147: float64 -> float16 -> float64 (RNE, overflow -> inf)."""
    with np.errstate(over="ignore"):
        return np.asarray(d, dtype=np.float64).astype(np.float16).astype(np.float64)


def _zero_points_vec(mu, d_eff, symmetric):
    """compute.py:162-166 (no +0.0 normalisation: the value only enters arithmetic here)."""
    if symmetric:
        return np.zeros_like(mu)
    r = mu / d_eff
    return np.clip(-np.copysign(np.floor(np.abs(r) + 0.5), r), -1.0, 1.0)


def ternary_blocks(y, variant="s", symmetric=True, kind="constant", constant=DEFAULT_SCALE_COEFF):
    """compute.py:169-201: grid-quantise (nb, n) coefficient rows.

    Returns (recon, codes int8, clamp bool, budget) where budget is the per-block grid bound
    of compute.py:246-249 (n*d^2/4, or (n/8)*sum(d_m^2)/4 for SS).
    """
    nb, n = y.shape
    mu = np.mean(y, axis=1)
    if variant == "s":
        d_raw = policy_scales(y, kind, constant)
        d16 = f16_round_cast(d_raw)
        d_eff = np.where(d16 > 0, d16, d_raw)
        z = _zero_points_vec(mu, d_eff, symmetric)[:, None]
        pre = round_half_away(y / d_eff[:, None]) + z
        codes = np.clip(pre, -1.0, 1.0)
        with np.errstate(invalid="ignore"):
            recon = d16[:, None] * (codes - z)
        return recon, codes.astype(np.int8), np.abs(pre) > 1.0, n * d16 ** 2 / 4.0
    m = n // SUB_BLOCKS
    subs = y.reshape(nb, SUB_BLOCKS, m)
    d_raw = policy_scales(subs.reshape(nb * SUB_BLOCKS, m), kind, constant).reshape(nb, SUB_BLOCKS)
    d16 = f16_round_cast(d_raw)
    d_eff = np.where(d16 > 0, d16, d_raw)
    mean_raw = np.mean(d_raw, axis=1)
    db = f16_round_cast(mean_raw)
    db = np.where(db > 0, db, mean_raw)
    z = _zero_points_vec(mu, db, symmetric)[:, None, None]
    pre = round_half_away(subs / d_eff[:, :, None]) + z
    codes = np.clip(pre, -1.0, 1.0)
    with np.errstate(invalid="ignore"):
        recon = (d16[:, :, None] * (codes - z)).reshape(nb, n)
    budget = m * np.sum(d16 ** 2, axis=1) / 4.0
    return recon, codes.reshape(nb, n).astype(np.int8), (np.abs(pre) > 1.0).reshape(nb, n), budget


def uniform3_blocks(blocks):
    """compute.py:204-211: per-block uniform 3-bit (7 steps over [min, max]); constant rows pass."""
    lo = blocks.min(axis=1, keepdims=True)
    hi = blocks.max(axis=1, keepdims=True)
    ok = hi > lo
    step = np.where(ok, (hi - lo) / 7.0, 1.0)
    rec = np.clip(step * np.floor(blocks / step + 0.5), lo, hi)
    return np.where(ok, rec, blocks)


class NonFiniteError(ValueError):
    """fwht_inverse's input check (transform.py:36-42 via _as_block), raised as DomainError there."""


def _check_inverse_input(ry):
    if not np.all(np.isfinite(ry)):
        raise NonFiniteError("fwht_inverse: input contains non-finite values")


def _report(a, blocks, y, recon, codes, clamp, budget, noro, size):
    """Shared tail of eval_error / eval_container (compute.py:241-269, 310-338)."""
    diff = recon - blocks
    err = diff.reshape(-1)[:size]
    wn = float(np.linalg.norm(a))
    block_err2 = np.sum(diff ** 2, axis=1)
    unclamped = ~clamp.any(axis=1)
    slack = float(np.min(budget[unclamped] - block_err2[unclamped])) if unclamped.any() else 0.0
    noro_err = (noro - blocks).reshape(-1)[:size]
    uni_err = (uniform3_blocks(blocks) - blocks).reshape(-1)[:size]
    return {"mse": float(np.mean(err ** 2)),
            "frobenius_rel": float(np.linalg.norm(err) / wn) if wn > 0 else 0.0,
            "linf_in": float(np.mean(np.max(np.abs(blocks), axis=1))),
            "linf_rot": float(np.mean(np.max(np.abs(y), axis=1))),
            "bound_slack": slack,
            "clamp_fraction": float(np.mean(clamp)),
            "zero_fraction": float(np.mean(codes == 0)),
            "mse_uniform3": float(np.mean(uni_err ** 2)),
            "mse_ternary_noro": float(np.mean(noro_err ** 2)),
            "n_blocks": int(blocks.shape[0]),
            "unclamped_blocks": int(np.sum(unclamped))}


def error_report(w, block_n=256, variant="s", symmetric=True, kind="constant", constant=DEFAULT_SCALE_COEFF):
    """eval_error (compute.py:221-269) -> dict of the ErrorReport fields."""
    a = np.asarray(w, dtype=np.float64)
    blocks, _ = blockify(a, block_n)
    y = fwht(blocks)
    ry, codes, clamp, budget = ternary_blocks(y, variant, symmetric, kind, constant)
    _check_inverse_input(ry)
    recon = fwht(ry)
    noro = ternary_blocks(blocks, variant, symmetric, kind, constant)[0]
    return _report(a, blocks, y, recon, codes, clamp, budget, noro, a.size)


def container_report(w, payload, n, variant, symmetric, kind="constant", constant=DEFAULT_SCALE_COEFF):
    """eval_container (compute.py:272-338): grid values from the payload, clamp re-derived."""
    a = np.asarray(w, dtype=np.float64)
    blocks, _ = blockify(a, n)
    y = fwht(blocks)
    ss = variant == "ss"
    quants, sb, zb, sub = split_payload(payload, n, ss)
    codes, _ = unpack_planes(quants, n)
    cf = codes.astype(np.float64)
    z = np.trunc(f16_value(zb))[:, None]
    if not ss:
        d16 = f16_value(sb)
        scales = d16[:, None]
        budget = n * d16 ** 2 / 4.0
    else:
        d16 = f16_value(sub)
        scales = np.repeat(d16, n // SUB_BLOCKS, axis=1)
        budget = (n // SUB_BLOCKS) * np.sum(d16 ** 2, axis=1) / 4.0
    ry = scales * (cf - z)
    _check_inverse_input(ry)
    pre = np.where(scales > 0, round_half_away(y / np.where(scales > 0, scales, 1.0)) + z, 2.0 * cf)
    clamp = np.abs(pre) > 1.0
    recon = fwht(ry)
    noro = ternary_blocks(blocks, variant, symmetric, kind, constant)[0]
    return _report(a, blocks, y, recon, codes, clamp, budget, noro, a.size)


def rotation_benefit(w, block_n=256, variant="s", symmetric=True, kind="constant", constant=DEFAULT_SCALE_COEFF):
    """compute.py:340-356: medians of the per-block MSEs of the three codecs."""
    a = np.asarray(w, dtype=np.float64)
    blocks, _ = blockify(a, block_n)
    ry = ternary_blocks(fwht(blocks), variant, symmetric, kind, constant)[0]
    _check_inverse_input(ry)
    rot = fwht(ry)
    noro = ternary_blocks(blocks, variant, symmetric, kind, constant)[0]
    uni = uniform3_blocks(blocks)
    med = lambda r: float(np.median(np.mean((r - blocks) ** 2, axis=1)))  # noqa: E731
    return {"rotated": med(rot), "unrotated": med(noro), "uniform3": med(uni)}


def pairwise_sum(v) -> float:
    """numpy's add.reduce over a contiguous float64 vector (numpy/_core/src/umath/loops_utils.h.src):
    n < 8 sequential; n <= 128 eight strided accumulators + tree + tail; else split at
    (n/2 rounded down to a multiple of 8) and recurse.  The GPU reduction replays this tree."""
    v = np.asarray(v, dtype=np.float64)

    def rec(lo, n):
        if n < 8:
            s = 0.0
            for i in range(n):
                s += float(v[lo + i])
            return s
        if n <= 128:
            r = [float(x) for x in v[lo:lo + 8]]
            i = 8
            while i < n - (n % 8):
                for k in range(8):
                    r[k] += float(v[lo + i + k])
                i += 8
            s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                s += float(v[lo + i])
                i += 1
            return s
        n2 = (n // 2) - (n // 2) % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)

    return 0.0 + rec(0, v.size)
