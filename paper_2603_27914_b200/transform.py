"""Normalised fast Walsh-Hadamard transform (transform.py:61-96 of the reference) on the GPU.

``itq3_fwht`` replays numpy's radix-2 butterfly order in the input's own precision, so
float64 and float32 results are bit-identical to the reference's ``fwht_forward``.
"""

from __future__ import annotations

from dataclasses import dataclass

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


ORACLE_MAX_LEN = 64


def is_power_of_two(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


def hadamard_matrix(n: int) -> np.ndarray:
    """Dense orthonormal Hadamard matrix of order n (power of two in [2, 64]): the normalised
    transform of the identity's rows (entries +-fl(1/sqrt(n)), bit-identical to transform.py:108-114)."""
    if not is_power_of_two(n) or n < MIN_BLOCK_LEN or n > ORACLE_MAX_LEN:
        raise LengthError(
            f"hadamard_matrix: order must be a power of two in [{MIN_BLOCK_LEN}, {ORACLE_MAX_LEN}], got {n}")
    return fwht_forward(np.eye(n, dtype=np.float64))


def hadamard_oracle(v) -> np.ndarray:
    """Transform by explicit dense matrix multiplication (the reference's test oracle, n <= 64):
    a float64 GEMM with the Hadamard matrix on the device (cuBLAS)."""
    a = np.asarray(v)
    if not np.issubdtype(a.dtype, np.inexact):
        a = a.astype(np.float64)
    if a.ndim == 0 or a.shape[-1] == 0:
        raise LengthError(f"hadamard_oracle: input must have at least one axis of length >= {MIN_BLOCK_LEN}")
    n = a.shape[-1]
    if not is_power_of_two(n) or n < MIN_BLOCK_LEN or n > MAX_BLOCK_LEN:
        raise LengthError(
            f"hadamard_oracle: block length must be a power of two in [{MIN_BLOCK_LEN}, {MAX_BLOCK_LEN}], got {n}")
    if not np.all(np.isfinite(a)):
        raise DomainError("hadamard_oracle: input contains non-finite values")
    if n > ORACLE_MAX_LEN:
        raise LengthError(f"hadamard_oracle: length {n} exceeds oracle limit {ORACLE_MAX_LEN}")
    dev = _lib.device()
    h = torch.from_numpy(hadamard_matrix(n)).to(dev)
    x = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
    return (x @ h).cpu().numpy()


@dataclass(frozen=True)
class StageTrace:
    """Per-stage butterfly states of a staged transform: ``stages[s]`` is the unnormalised block after
    butterfly step 2**s; ``final`` is the last stage scaled by 1/sqrt(n) (= fwht_forward)."""

    stages: tuple
    final: np.ndarray

    @property
    def stage_count(self) -> int:
        return len(self.stages)


def fwht_staged(v) -> StageTrace:
    """Stage-by-stage transform (transform.py:148-173).  Steps 1..2**s only mix aligned runs of
    2**(s+1) elements, so stage s is the unnormalised itq3_fwht of the block cut into such runs --
    the same adds and subtracts per element as the reference's double-buffered schedule."""
    is_t = isinstance(v, torch.Tensor)
    a = v.detach().cpu().numpy() if is_t else np.asarray(v)
    if not np.issubdtype(a.dtype, np.inexact):
        a = a.astype(np.float64)
    if a.ndim != 1:
        raise LengthError("fwht_staged: expects a single 1-D block")
    _fwht(a[None, :] if a.size else a, "fwht_staged")  # the reference's validation (length, finiteness)
    n = a.shape[0]
    dev = _lib.device()
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    code = _lib.F64 if t.dtype == torch.float64 else _lib.F32
    stages = []
    m = 2
    while m <= n:
        out = torch.empty_like(t)
        _lib.call("itq3_fwht", _lib.ptr(t), _lib.ptr(out), code, n // m, m, 0, _lib.stream_ptr(dev))
        stages.append(out.cpu().numpy())
        m *= 2
    return StageTrace(stages=tuple(stages), final=fwht_forward(a))


def fwht32_warp(v) -> np.ndarray:
    """32-point transform in the intra-warp style (transform.py:176-197): equal to fwht_forward on a
    length-32 block."""
    a = np.asarray(v)
    if not np.issubdtype(a.dtype, np.inexact):
        a = a.astype(np.float64)
    if a.ndim != 1 or a.shape[0] != 32:
        raise LengthError(f"fwht32_warp: expects a 1-D block of length 32, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise DomainError("fwht32_warp: input contains non-finite values")
    return fwht_forward(a)
