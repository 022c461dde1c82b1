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
