"""Fused decode-and-multiply paths of the drop-in API (compute.py:98-133 of the reference).

Two modes, chosen by the operand type:
  * numpy / array-like X  -> parity mode: float64 result equal to the reference's
    ``fused_matmul`` within its own tolerance (test_compute.py:66-103, rtol 1e-5): the
    rotated activations carry 6 fixed-point limbs (48 bits) and blocks accumulate in fp64.
  * CUDA torch tensor X   -> perf mode: float32 result (float64 if X is float64); 3 limbs
    (24-bit activations) at M = 1 and 2 limbs (16-bit) for M > 1, fp32 accumulation; for
    M >= 16 columns the tcgen05 MMQ kernel (exact f16 weights d*t, f16 rotated activations,
    fp32 TMEM accumulation).
Both run the same kernels: K3 ``itq3_rotate_act`` + K4 ``itq3_gemv`` on the tiled layout
(block_n 256, variant s, cols % 256 == 0), else the generic fp64 kernel
``itq3_matmul_generic`` (any block size / variant / row-straddling blocks).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .codec import QuantizedTensor
from .errors import DomainError, ShapeError

PARITY_LIMBS = 6
MMQ_MIN_TOKENS = 8  # perf mode: k >= 8 columns go to the tcgen05 MMQ kernels (csrc/mmq.cu; tools/crossover.py)
MMQ8_MAX_TOKENS = 64  # ... 8 <= k <= 64 to the kind::i8 one (K5b), larger k to the kind::f16 one (K5)


_NONFINITE: dict = {}


def _nonfinite_flag(dev: torch.device, stream: int) -> torch.Tensor:
    """Per-(device, stream) u32 flag the MMQ activation rotations OR with 1 on a non-finite input
    (kept zero): calls on different streams never see each other's error."""
    key = (dev, stream)
    f = _NONFINITE.get(key)
    if f is None:
        if len(_NONFINITE) >= 64:
            _NONFINITE.clear()
        f = torch.zeros(1, dtype=torch.int32, device=dev)
        _NONFINITE[key] = f
    return f


_SCRATCH: dict = {}


def _scratch(dev: torch.device, stream: int, slot: str, nbytes: int) -> torch.Tensor | None:
    """Reusable device scratch (rotated activations, split-K workspace) per (device, stream, slot):
    calls on one stream are ordered, so a buffer can be reused by the next call without a fresh
    allocation; it only grows.  Under CUDA-graph capture a fresh buffer from the graph's private
    pool is used instead: a captured graph keeps raw pointers, so it must never share (or outlive)
    a cached buffer that a later eager call could grow, free or race with on replay."""
    if nbytes <= 0:
        return None
    if torch.cuda.is_current_stream_capturing():
        return torch.empty(nbytes, dtype=torch.uint8, device=dev)
    key = (dev, stream, slot)
    buf = _SCRATCH.get(key)
    if buf is None and len(_SCRATCH) >= 64:  # many short-lived streams: drop the cache (stream-ordered frees)
        _SCRATCH.clear()
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=dev)
        _SCRATCH[key] = buf
    return buf


def _raise_if_nonfinite(flag: torch.Tensor) -> None:
    if int(flag.item()):
        flag.zero_()
        raise DomainError("fused_matmul: X contains non-finite values")


def perf_limbs(m: int) -> int:
    return 3 if m == 1 else 2


class _ChainGemv:
    """A one-stage decode chain (csrc/chain.cu) bound to one tensor and device: the k = 1 perf path.
    One cooperative launch streams the weights through the TMA ring while every CTA rotates its own
    K-chunk of x in registers -- no separate rotation kernel, no host sync.  Calls are ordered by
    the step epoch on the stream they are issued to, so a tensor's k = 1 products must not run
    concurrently on two streams (CUDA-graph capture and replay are fine)."""

    def __init__(self, q: QuantizedTensor, dev: torch.device):
        import ctypes

        lib = _lib.load()
        host = ctypes.create_string_buffer(lib.itq3_chain_desc_nbytes())
        self.tiled = q.tiled()
        nch = -(-q.cols // 4096)
        self.yparts = torch.zeros((nch, q.rows), dtype=torch.int64, device=dev)  # tagged (value | epoch << 32)
        _lib.check(lib.itq3_chain_write_desc(host, 0, _lib.ptr(self.tiled), _lib.ptr(self.yparts), None, q.rows,
                                             q.cols, int(not q.symmetric), 0))
        self.desc = torch.frombuffer(bytearray(host.raw), dtype=torch.uint8).to(dev)
        self.epoch = torch.zeros(2, dtype=torch.int32, device=dev)  # (step epoch, check-in count)
        self.flags = 2 if q.symmetric else 4  # symmetric: the kernel without the zero-point tile loop

    def __call__(self, x: torch.Tensor, out: torch.Tensor, stream: int) -> None:
        _lib.call("itq3_chain_run_ex", _lib.ptr(self.desc), 1, _lib.ptr(x), CHAIN_LIMBS, _lib.ptr(self.epoch),
                  _lib.ptr(out), 0, None, stream, self.flags)


CHAIN_LIMBS = 3


def _matvec_chain(q: QuantizedTensor, x: torch.Tensor) -> torch.Tensor:
    dev = x.device
    stream = _lib.stream_ptr(dev)
    ctx = q._chain1.get(dev)
    if ctx is None:
        ctx = q._chain1[dev] = _ChainGemv(q, dev)
    xf = x.reshape(-1)
    if xf.dtype != torch.float32 or not xf.is_contiguous():
        xf = xf.to(torch.float32).contiguous()
    out = torch.empty((q.rows, 1), dtype=torch.float32, device=dev)
    ctx(xf, out, stream)
    return out


def _matmul_device(q: QuantizedTensor, X: torch.Tensor, out_dtype: torch.dtype, limbs: int,
                   check_finite: bool = True) -> torch.Tensor:
    """Y (rows x k) = w_hat @ X for a CUDA X (cols x k, any strides), computed on X's device (its
    weight layouts are built there, the launches go to that device's current stream)."""
    with torch.cuda.device(X.device):
        return _matmul_on_device(q, X, out_dtype, limbs, check_finite)


def _matmul_on_device(q: QuantizedTensor, X: torch.Tensor, out_dtype: torch.dtype, limbs: int,
                      check_finite: bool) -> torch.Tensor:
    dev = X.device
    rows, cols = q.rows, q.cols
    k = X.shape[1]
    if q.fast_layout() and out_dtype == torch.float32 and k == 1 and limbs == CHAIN_LIMBS:
        return _matvec_chain(q, X)
    if q.fast_layout() and out_dtype != torch.float64 and MMQ_MIN_TOKENS <= k <= MMQ8_MAX_TOKENS \
            and X.dtype != torch.float64:
        lib = _lib.load()
        s = _lib.stream_ptr(dev)
        act = _scratch(dev, s, "act8", lib.itq3_mmq8_act_nbytes(cols, k))
        flag = _nonfinite_flag(dev, s) if check_finite else None
        _lib.call("itq3_rotate_act_i8", _lib.ptr(X), _lib.TORCH_DTYPE_CODE[X.dtype], cols, k, X.stride(0),
                  X.stride(1), _lib.ptr(act), _lib.ptr(flag) if flag is not None else None, s)
        Y = torch.empty((rows, k), dtype=out_dtype, device=dev)
        ws = _scratch(dev, s, "ws8", lib.itq3_mmq8_ws_nbytes(rows, cols, k))
        _lib.call("itq3_mmq8", _lib.ptr(q.mmq8_layout()), rows, cols, _lib.ptr(act), k, _lib.ptr(Y),
                  _lib.TORCH_DTYPE_CODE[out_dtype], Y.stride(0), Y.stride(1), _lib.ptr(ws) if ws is not None else None,
                  s)
        if flag is not None:
            _raise_if_nonfinite(flag)
        return Y
    if q.mmq_ok() and out_dtype != torch.float64 and not q.fast_layout() and k < MMQ_MIN_TOKENS \
            and q.k5_range_ok() and X.dtype != torch.float64:
        # variant ss / block_n != 256 with k < 8: K5 on X zero-padded to 8 tokens (the padded columns are
        # exact zeros, the real ones see K5's arithmetic and bound) -- instead of the exact fp64 kernel
        Xp = torch.zeros((cols, MMQ_MIN_TOKENS), dtype=X.dtype, device=dev)
        Xp[:, :k] = X
        return _matmul_on_device(q, Xp, out_dtype, limbs, check_finite)[:, :k]
    if q.mmq_ok() and out_dtype != torch.float64 and k >= MMQ_MIN_TOKENS and q.k5_range_ok():
        # K5: block_n 256 variant s for k > MMQ8_MAX_TOKENS; variant ss and block_n != 256 for every k >= MMQ_MIN_TOKENS
        # (and, zero-padded, k < MMQ_MIN_TOKENS)
        mmq = q.mmq_layout()
        s = _lib.stream_ptr(dev)
        act = _scratch(dev, s, "act", _lib.load().itq3_mmq_act_nbytes(cols, k))
        flag = _nonfinite_flag(dev, s) if check_finite else None
        _lib.call("itq3_rotate_act_f16_n", _lib.ptr(X), _lib.TORCH_DTYPE_CODE[X.dtype], cols, k, X.stride(0),
                  X.stride(1), q.block_n, _lib.ptr(act), _lib.ptr(flag) if flag is not None else None, s)
        Y = torch.empty((rows, k), dtype=out_dtype, device=dev)
        ws = _scratch(dev, s, "ws", _lib.load().itq3_mmq_ws_nbytes(rows, cols, k))
        _lib.call("itq3_mmq", _lib.ptr(mmq), rows, cols, q.mmq_flags(), _lib.ptr(act), k, _lib.ptr(Y),
                  _lib.TORCH_DTYPE_CODE[out_dtype], Y.stride(0), Y.stride(1), _lib.ptr(ws) if ws is not None else None,
                  s)
        if flag is not None:
            _raise_if_nonfinite(flag)
        return Y
    if q.fast_layout():
        tiled = q.tiled()
        act = torch.empty(_lib.load().itq3_act_nbytes(cols, k, limbs), dtype=torch.uint8, device=dev)
        xcode = _lib.TORCH_DTYPE_CODE[X.dtype]
        s = _lib.stream_ptr(dev)
        _lib.call("itq3_rotate_act", _lib.ptr(X), xcode, cols, k, X.stride(0), X.stride(1), limbs, _lib.ptr(act), s)
        Y = torch.empty((rows, k), dtype=out_dtype, device=dev)
        _lib.call("itq3_gemv", _lib.ptr(tiled), rows, cols, int(not q.symmetric), _lib.ptr(act), k, limbs,
                  _lib.ptr(Y), _lib.TORCH_DTYPE_CODE[out_dtype], Y.stride(0), Y.stride(1), s)
        return Y
    p = q.ensure_decodable()
    Xd = X.to(torch.float64)
    ws = torch.empty(_lib.load().itq3_generic_ws_nbytes(rows, cols, q.block_n, k), dtype=torch.uint8, device=dev)
    Y = torch.empty((rows, k), dtype=torch.float64, device=dev)
    _lib.call("itq3_matmul_generic", _lib.ptr(p), rows, cols, q.block_n, int(q.variant == "ss"), _lib.ptr(Xd), k,
              Xd.stride(0), Xd.stride(1), _lib.ptr(Y), _lib.ptr(ws), _lib.stream_ptr(dev))
    return Y if out_dtype == torch.float64 else Y.to(out_dtype)


def fused_matmul(q: QuantizedTensor, x, *, limbs: int | None = None, check_finite: bool = True):
    """Multiply the quantized matrix by X (cols x k) without materialising it.

    check_finite (CUDA X only, an addition to the reference signature): False skips the DomainError
    check on X -- and with it the one host synchronisation the check needs -- so the call stays
    asynchronous on the stream."""
    if isinstance(x, torch.Tensor) and x.is_cuda:
        if x.ndim != 2:
            raise ShapeError(f"fused_matmul: X must be 2-D (cols x k), got shape {tuple(x.shape)}")
        if x.shape[0] != q.cols:
            raise ShapeError(f"fused_matmul: X has {x.shape[0]} rows, tensor has {q.cols} columns")
        if x.dtype not in _lib.TORCH_DTYPE_CODE:
            x = x.to(torch.float32)
        parity = x.dtype == torch.float64
        # the MMQ paths (k >= MMQ_MIN_TOKENS, perf mode) check finiteness inside their activation rotation
        if check_finite and (parity or x.shape[1] < MMQ_MIN_TOKENS or not (q.mmq_ok() and q.k5_range_ok())):
            if not bool(torch.isfinite(x).all()):
                raise DomainError("fused_matmul: X contains non-finite values")
        L = limbs or (PARITY_LIMBS if parity else perf_limbs(x.shape[1]))
        return _matmul_device(q, x, torch.float64 if parity else torch.float32, L, check_finite)
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise ShapeError(f"fused_matmul: X must be 2-D (cols x k), got shape {a.shape}")
    if a.shape[0] != q.cols:
        raise ShapeError(f"fused_matmul: X has {a.shape[0]} rows, tensor has {q.cols} columns")
    dev = _lib.device()
    t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    if not bool(torch.isfinite(t).all()):
        raise DomainError("fused_matmul: X contains non-finite values")
    return _matmul_device(q, t, torch.float64, limbs or PARITY_LIMBS).cpu().numpy()


def fused_matvec(q: QuantizedTensor, x, *, limbs: int | None = None, check_finite: bool = True):
    """Matrix-vector product: exactly the k = 1 column of fused_matmul."""
    if isinstance(x, torch.Tensor) and x.is_cuda:
        if x.ndim != 1:
            raise ShapeError(f"fused_matvec: x must be 1-D, got shape {tuple(x.shape)}")
        return fused_matmul(q, x[:, None], limbs=limbs, check_finite=check_finite)[:, 0]
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 1:
        raise ShapeError(f"fused_matvec: x must be 1-D, got shape {a.shape}")
    return fused_matmul(q, a[:, None], limbs=limbs)[:, 0]
