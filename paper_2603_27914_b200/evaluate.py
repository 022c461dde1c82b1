"""Evaluation harness of the drop-in API -- eval_error / eval_container / rotation_benefit /
ablate_block_size and their report types (reference pkg/src/itq3/compute.py:31-400).

SURVEY.md §8(f)2: the reference measures eps_q with a vectorised numpy encoder at ~15-35 us per
block (plus the two baselines); here one K8 launch (``itq3_eval``, csrc/eval.cu) quantises every
block, reconstructs it, runs both baselines and reduces the report on the device.  Every field
is bit-exact with the reference except ``frobenius_rel`` (the reference's norm is a BLAS ddot,
whose summation order is not numpy's; equal to rounding).

``generate_weights`` is the reference's seeded synthetic-input generator (numpy PCG64 streams,
compute.py:58-95); it produces inputs, not results, and stays on the host so seeds give the
same matrices as the reference.
"""

from __future__ import annotations

import csv
import io
import json
import math
from dataclasses import asdict, dataclass

import numpy as np
import torch

from . import _lib
from .codec import BLOCK_SIZES, QuantConfig, QuantizedTensor, _weights_on_device
from .errors import DomainError, ShapeError
from .quantizer import POLICY_CODE, ScalePolicy

DISTRIBUTIONS = ("gaussian", "laplace", "student-t", "outlier")

# itq3_eval_field (include/itq3.h)
_ERR2, _NORO2, _UNI2 = 6, 7, 8


@dataclass(frozen=True)
class ErrorReport:
    """Reconstruction error metrics for one quantization configuration (compute.py:31-45)."""

    mse: float
    frobenius_rel: float
    linf_in: float
    linf_rot: float
    bound_slack: float
    clamp_fraction: float
    zero_fraction: float
    mse_uniform3: float
    mse_ternary_noro: float
    n_blocks: int
    unclamped_blocks: int


@dataclass(frozen=True)
class AblationRow:
    """One block-size sweep entry: error plus transform flops per weight (compute.py:48-54)."""

    block_n: int
    mse: float
    relative_overhead: float


def generate_weights(dist: str, rows: int, cols: int, seed: int, nu: float = 3.0, outlier_frac: float = 0.01,
                     outlier_mult: float = 20.0) -> np.ndarray:
    """Seeded synthetic weight matrix (compute.py:58-95): same generators, seeds and errors."""
    if dist not in DISTRIBUTIONS:
        raise DomainError(f"generate_weights: unknown distribution {dist!r}, expected one of {DISTRIBUTIONS}")
    if rows <= 0 or cols <= 0:
        raise DomainError(f"generate_weights: dims must be positive, got {rows}x{cols}")
    rng = np.random.default_rng(seed)
    if dist == "gaussian":
        return rng.standard_normal((rows, cols))
    if dist == "laplace":
        return rng.laplace(size=(rows, cols))
    if dist == "student-t":
        if not (nu > 0 and math.isfinite(nu)):
            raise DomainError(f"generate_weights: nu must be positive and finite, got {nu}")
        return rng.standard_t(nu, size=(rows, cols))
    if not 0.0 <= outlier_frac <= 1.0:
        raise DomainError(f"generate_weights: outlier fraction must be in [0, 1], got {outlier_frac}")
    if not math.isfinite(outlier_mult):
        raise DomainError(f"generate_weights: outlier multiplier must be finite, got {outlier_mult}")
    w = rng.standard_normal((rows, cols))
    k = int(round(outlier_frac * w.size))
    if k:
        idx = rng.choice(w.size, size=k, replace=False)
        w.reshape(-1)[idx] *= outlier_mult
    return w


def _shape_of(w) -> tuple:
    return tuple(w.shape) if isinstance(w, torch.Tensor) else np.shape(w)


class _EvalRun:
    """One itq3_eval launch; keeps the workspace so per-block fields can be read afterwards."""

    def __init__(self, t: torch.Tensor, block_n: int, ss: bool, policy: ScalePolicy, symmetric: bool,
                 payload: torch.Tensor | None):
        self.nb = -(-t.numel() // block_n)
        self.n = block_n
        lib = _lib.load()
        self.ws = torch.empty(lib.itq3_eval_ws_nbytes(self.nb, block_n), dtype=torch.uint8, device=t.device)
        self.report = torch.empty(12, dtype=torch.float64, device=t.device)
        dtype = _lib.F32 if t.dtype == torch.float32 else _lib.F64
        _lib.call("itq3_eval", _lib.ptr(t), dtype, t.numel(), block_n, int(ss), POLICY_CODE[policy.kind],
                  policy.coefficient(), int(symmetric), 0 if payload is None else _lib.ptr(payload),
                  _lib.ptr(self.ws), _lib.ptr(self.report), _lib.stream_ptr(t.device))

    def field(self, f: int) -> torch.Tensor:
        off = _lib.load().itq3_eval_ws_offset(self.nb, self.n, f)
        return self.ws[off:off + 8 * self.nb].view(torch.float64)

    def check_finite(self, r=None) -> None:
        r = self.report.cpu().tolist() if r is None else r
        if r[11]:
            raise DomainError("fwht_inverse: input contains non-finite values")

    def to_report(self) -> ErrorReport:
        r = self.report.cpu().tolist()
        self.check_finite(r)
        return ErrorReport(mse=r[0], frobenius_rel=r[1], linf_in=r[2], linf_rot=r[3], bound_slack=r[4],
                           clamp_fraction=r[5], zero_fraction=r[6], mse_uniform3=r[7], mse_ternary_noro=r[8],
                           n_blocks=int(r[9]), unclamped_blocks=int(r[10]))


def _checked_device_weights(w, who: str, what: str) -> torch.Tensor:
    t = _weights_on_device(w, _lib.device())
    if not bool(torch.isfinite(t).all()):
        raise DomainError(f"{who}: {what} contains non-finite values")
    return t


def eval_error(w, cfg: QuantConfig | None = None) -> ErrorReport:
    """Quantize, decode and measure error against the two baselines (compute.py:221-269)."""
    cfg = cfg or QuantConfig()
    shape = _shape_of(w)
    if len(shape) != 2 or 0 in shape:
        raise ShapeError(f"eval_error: expected a non-empty 2-D matrix, got shape {shape}")
    t = _checked_device_weights(w, "eval_error", "input")
    return _EvalRun(t, cfg.block_n, cfg.variant == "ss", cfg.policy, cfg.symmetric, None).to_report()


def eval_container(w, q: QuantizedTensor, policy: ScalePolicy | None = None) -> ErrorReport:
    """Error report of a stored tensor against its reference weights (compute.py:272-338)."""
    policy = policy or ScalePolicy()
    shape = _shape_of(w)
    if len(shape) != 2 or shape != (q.rows, q.cols):
        raise ShapeError(f"eval_container: reference shape {shape} does not match tensor {q.rows}x{q.cols}")
    t = _checked_device_weights(w, "eval_container", "reference")
    nb = -(-q.rows * q.cols // q.block_n)
    payload = q.ensure_decodable()
    if payload.shape[0] != nb:
        raise ShapeError(f"eval_container: container has {payload.shape[0]} blocks, reference needs {nb}")
    if payload.device != t.device:
        payload = payload.to(t.device)
    return _EvalRun(t, q.block_n, q.variant == "ss", policy, q.symmetric, payload).to_report()


def _median(v: torch.Tensor) -> float:
    """np.median: middle order statistic, or the mean of the two middle ones."""
    s, _ = torch.sort(v)
    n = s.numel()
    if n % 2:
        return float(s[n // 2].item())
    return float(((s[n // 2 - 1] + s[n // 2]) / 2.0).item())


def rotation_benefit(w, cfg: QuantConfig | None = None) -> dict[str, float]:
    """Median per-block MSE of the rotated codec vs the two baselines (compute.py:340-356)."""
    cfg = cfg or QuantConfig()
    shape = _shape_of(w)
    if len(shape) != 2 or 0 in shape:
        raise ShapeError(f"rotation_benefit: expected a non-empty 2-D matrix, got shape {shape}")
    t = _weights_on_device(w, _lib.device())
    run = _EvalRun(t, cfg.block_n, cfg.variant == "ss", cfg.policy, cfg.symmetric, None)
    run.check_finite()
    n = float(cfg.block_n)
    return {"rotated": _median(run.field(_ERR2) / n),
            "unrotated": _median(run.field(_NORO2) / n),
            "uniform3": _median(run.field(_UNI2) / n)}


def ablate_block_size(sweep=(32, 64, 128, 256), dist: str = "outlier", rows: int = 32, cols: int = 512,
                      base_seed: int = 0, replicates: int = 9, cfg: QuantConfig | None = None, nu: float = 3.0,
                      outlier_frac: float = 0.01, outlier_mult: float = 20.0) -> list[AblationRow]:
    """Block-size sweep over shared-seed tensors (compute.py:359-400)."""
    sizes = tuple(sweep)
    for n in sizes:
        if n not in BLOCK_SIZES:
            raise DomainError(f"ablate_block_size: block_n {n} not in {BLOCK_SIZES}")
    if replicates <= 0:
        raise DomainError(f"ablate_block_size: replicates must be positive, got {replicates}")
    cfg = cfg or QuantConfig()
    tensors = [generate_weights(dist, rows, cols, base_seed + t, nu=nu, outlier_frac=outlier_frac,
                                outlier_mult=outlier_mult) for t in range(replicates)]
    dev = [_weights_on_device(w, _lib.device()) for w in tensors]
    out = []
    for n in sizes:
        ncfg = QuantConfig(block_n=n, variant=cfg.variant, policy=cfg.policy, symmetric=cfg.symmetric)
        mses = [eval_error(t, ncfg).mse for t in dev]
        out.append(AblationRow(block_n=n, mse=float(np.median(mses)), relative_overhead=math.log2(n) + 1))
    return out


def _rows(obj) -> list[dict]:
    if isinstance(obj, (ErrorReport, AblationRow)):
        return [asdict(obj)]
    return [asdict(r) for r in obj]


def report_json(obj) -> str:
    """An ErrorReport (object) or a sequence of AblationRows (list) as indented JSON."""
    rows = _rows(obj)
    return json.dumps(rows[0] if isinstance(obj, (ErrorReport, AblationRow)) else rows, indent=2)


def report_csv(obj) -> str:
    """Report rows as CSV with the field names as header."""
    rows = _rows(obj)
    buf = io.StringIO()
    writer = csv.DictWriter(buf, fieldnames=list(rows[0].keys()), lineterminator="\n")
    writer.writeheader()
    writer.writerows(rows)
    return buf.getvalue()
