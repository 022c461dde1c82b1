"""Normalised fast Walsh-Hadamard transform (transform.py:61-96 of the reference) on the GPU.

``itq3_fwht`` replays numpy's radix-2 butterfly order in the input's own precision, so
float64 and float32 results are bit-identical to the reference's ``fwht_forward``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import DomainError, LengthError

MAX_BLOCK_LEN = 512
MIN_BLOCK_LEN = 2


def _fwht(v, op: str):
    is_t = isinstance(v, torch.Tensor)
    a = v if is_t else np.asarray(v)
    if not is_t and not np.issubdtype(a.dtype, np.inexact):
        a = a.astype(np.float64)
    if a.ndim == 0 or a.shape[-1] == 0:
        raise LengthError(f"{op}: input must have at least one axis of length >= {MIN_BLOCK_LEN}")
    n = a.shape[-1]
    if n < MIN_BLOCK_LEN or n > MAX_BLOCK_LEN or n & (n - 1):
        raise LengthError(f"{op}: block length must be a power of two in [{MIN_BLOCK_LEN}, {MAX_BLOCK_LEN}], got {n}")
    dev = _lib.device()
    if is_t:
        t = a.to(dev)
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
    else:
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    t = t.contiguous()
    if not bool(torch.isfinite(t).all()):
        raise DomainError(f"{op}: input contains non-finite values")
    out = torch.empty_like(t)
    code = _lib.F64 if t.dtype == torch.float64 else _lib.F32
    _lib.call("itq3_fwht", _lib.ptr(t), _lib.ptr(out), code, t.numel() // n, n, 1, _lib.stream_ptr(dev))
    return out if is_t else out.cpu().numpy()


def fwht_forward(v):
    """Normalised WHT along the last axis (same shape and dtype; input untouched)."""
    return _fwht(v, "fwht_forward")


def fwht_inverse(v):
    """Inverse transform (identical to the forward one: H/sqrt(n) is an involution)."""
    return _fwht(v, "fwht_inverse")
