"""Scale policy and ternary grid types of the drop-in API.

The arithmetic of the scale rules runs inside the K1 encoder kernel (csrc/codec.cu,
``encode_kernel``); this module only carries the configuration objects and constants
the reference exposes (pkg/src/itq3/quantizer.py:24-75).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import DomainError

DEFAULT_SCALE_COEFF = 0.7979  # E|x| of a unit Gaussian as stored by the reference (quantizer.py:24)
EPSILON_D = 1e-8  # degenerate-block scale floor (quantizer.py:28)
POLICY_KINDS = ("constant", "argmin", "mean-abs")

# Grid minimiser of the Gaussian ternary MSE over alpha = k * 1e-3, k = 1..2000 (quantizer.py:130-138).
# The reference recomputes it with scipy quadrature at first use; the value (k = 878) is pinned
# against the reference in tests/test_oracle_golden.py, so the product carries the constant.
ARGMIN_SCALE_COEFF = float.fromhex("0x1.c189374bc6a7fp-1")

POLICY_CODE = {"constant": 0, "argmin": 1, "mean-abs": 2}


def argmin_scale_coeff() -> float:
    """Coefficient of the "argmin" policy (0.878)."""
    return ARGMIN_SCALE_COEFF


@dataclass(frozen=True)
class ScalePolicy:
    """Per-block ternary scale rule: constant * sigma, argmin * sigma, or (2/3) mean |y|."""

    kind: str = "constant"
    constant: float = DEFAULT_SCALE_COEFF

    def __post_init__(self):
        if self.kind not in POLICY_KINDS:
            raise DomainError(f"ScalePolicy: unknown kind {self.kind!r}, expected one of {POLICY_KINDS}")
        if not (self.constant > 0 and math.isfinite(self.constant)):
            raise DomainError(f"ScalePolicy: constant must be positive and finite, got {self.constant}")

    def coefficient(self) -> float:
        return ARGMIN_SCALE_COEFF if self.kind == "argmin" else float(self.constant)


@dataclass(frozen=True)
class TernaryGrid:
    """Reconstruction grid d * (q - z), q in {-1, 0, 1}."""

    d: float
    z: int = 0

    def __post_init__(self):
        if not (self.d > 0 and math.isfinite(self.d)):
            raise DomainError(f"TernaryGrid: scale must be positive and finite, got {self.d}")
        if self.z not in (-1, 0, 1):
            raise DomainError(f"TernaryGrid: zero-point must be -1, 0, or 1, got {self.z}")


# ------------------------------------------------------------------------------------------------
# Block utilities (quantizer.py:78-197 of the reference): computed by csrc/util.cu on the device in
# float64 with the reference's data flow; the scalar rules (optimal_scale, ternary_mse) are plain
# float arithmetic, as in the reference.
# ------------------------------------------------------------------------------------------------
@dataclass(frozen=True)
class BlockStats:
    """Statistics of one block: size, mean, population sigma, l1 and linf norms, excess kurtosis."""

    n: int
    mean: float
    sigma: float
    l1: float
    linf: float
    excess_kurtosis: float


def _device_f64(x, op: str):
    import numpy as np
    import torch

    from . import _lib

    a = np.asarray(x, dtype=np.float64)
    if not np.all(np.isfinite(a)):
        raise DomainError(f"{op}: input contains non-finite values")
    dev = _lib.device()
    return a, torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).to(dev), dev


def block_stats(v) -> BlockStats:
    """Population statistics of one block (one device launch, numpy's summation order)."""
    import numpy as np
    import torch

    from . import _lib

    a = np.asarray(v, dtype=np.float64)
    if a.ndim != 1 or a.size == 0:
        raise DomainError("block_stats: expects a non-empty 1-D block")
    _, t, dev = _device_f64(a, "block_stats")
    out = torch.empty(6, dtype=torch.float64, device=dev)
    _lib.call("itq3_block_stats", _lib.ptr(t), a.size, _lib.ptr(out), _lib.stream_ptr(dev))
    n, mean, sigma, l1, linf, kurt = out.cpu().tolist()
    return BlockStats(n=int(n), mean=mean, sigma=sigma, l1=l1, linf=linf, excess_kurtosis=kurt)


def ternary_mse(alpha: float, sigma: float) -> float:
    """Gaussian MSE of the dead-zone ternary quantiser with threshold and level alpha (values with
    |x| <= alpha map to 0, the others to +-alpha), x ~ N(0, sigma^2).  Closed form of the reference's two
    quadratures (quantizer.py:102-127; agreement ~1e-12, the reference's own tolerance is 1e-9):
    with a = alpha / sigma, Phi the normal CDF, phi the density, Q = 1 - Phi,
    mse / sigma^2 = 2 [(Phi(a) - 1/2 - a phi(a)) + ((1 + a^2) Q(a) - a phi(a))]."""
    if not (alpha > 0 and math.isfinite(alpha)):
        raise DomainError(f"ternary_mse: alpha must be positive and finite, got {alpha}")
    if not (sigma > 0 and math.isfinite(sigma)):
        raise DomainError(f"ternary_mse: sigma must be positive and finite, got {sigma}")
    a = alpha / sigma
    phi = math.exp(-0.5 * a * a) / math.sqrt(2.0 * math.pi)
    dead = 0.5 * math.erf(a / math.sqrt(2.0)) - a * phi
    tail = (1.0 + a * a) * 0.5 * math.erfc(a / math.sqrt(2.0)) - a * phi
    return 2.0 * sigma * sigma * (dead + tail)


def optimal_scale(stats: BlockStats, policy: ScalePolicy) -> float:
    """Block scale chosen by `policy` from the block's statistics, never below EPSILON_D
    (quantizer.py:141-149)."""
    if policy.kind == "constant":
        d = policy.constant * stats.sigma
    elif policy.kind == "argmin":
        d = argmin_scale_coeff() * stats.sigma
    else:
        d = (2.0 / 3.0) * (stats.l1 / stats.n)
    return d if d > 0 else EPSILON_D


def ternary_quantize(x, grid: TernaryGrid):
    """Codes of x on the grid (device kernel): x / d rounded half away from zero, shifted by z and
    clipped to [-1, 1]; int8 array for array input, int for a scalar."""
    import numpy as np
    import torch

    from . import _lib

    a, t, dev = _device_f64(x, "ternary_quantize")
    out = torch.empty(t.numel(), dtype=torch.int8, device=dev)
    _lib.call("itq3_ternary_quantize", _lib.ptr(t), t.numel(), float(grid.d), int(grid.z), _lib.ptr(out),
              _lib.stream_ptr(dev))
    codes = out.cpu().numpy().reshape(a.shape)
    if np.isscalar(x) or np.ndim(x) == 0:
        return int(codes)
    return codes


def ternary_dequantize(code, grid: TernaryGrid):
    """Grid values d (code - z) of integer codes in [-1, 1] (device kernel)."""
    import numpy as np
    import torch

    from . import _lib

    c = np.asarray(code)
    if not np.issubdtype(c.dtype, np.integer):
        raise DomainError("ternary_dequantize: codes must be integers")
    if c.size and (c.min() < -1 or c.max() > 1):
        raise DomainError("ternary_dequantize: codes must lie in {-1, 0, 1}")
    dev = _lib.device()
    t = torch.from_numpy(np.ascontiguousarray(c, dtype=np.int8).reshape(-1)).to(dev)
    out = torch.empty(t.numel(), dtype=torch.float64, device=dev)
    _lib.call("itq3_ternary_dequantize", _lib.ptr(t), t.numel(), float(grid.d), int(grid.z), _lib.ptr(out),
              _lib.stream_ptr(dev))
    res = out.cpu().numpy().reshape(c.shape)
    if np.isscalar(code) or np.ndim(code) == 0:
        return float(res)
    return res


def uniform_quantize(x, bits: int, wmin: float, wmax: float):
    """The b-bit uniform baseline on [wmin, wmax]: nearest multiple of (wmax - wmin) / (2^b - 1),
    clamped to the range (device kernel)."""
    import numpy as np
    import torch

    from . import _lib

    if not 2 <= int(bits) <= 8:
        raise DomainError(f"uniform_quantize: bits must be in [2, 8], got {bits}")
    if not (wmin < wmax):
        raise DomainError(f"uniform_quantize: need wmin < wmax, got [{wmin}, {wmax}]")
    a, t, dev = _device_f64(x, "uniform_quantize")
    delta = (wmax - wmin) / (2 ** int(bits) - 1)
    out = torch.empty(t.numel(), dtype=torch.float64, device=dev)
    _lib.call("itq3_uniform_quantize", _lib.ptr(t), t.numel(), float(delta), float(wmin), float(wmax),
              _lib.ptr(out), _lib.stream_ptr(dev))
    res = out.cpu().numpy().reshape(a.shape)
    if np.isscalar(x) or np.ndim(x) == 0:
        return float(res)
    return res
