"""B200-native ITQ3_S hot path: drop-in for the reference ``itq3`` quantize / pack /
dequantize / fused-matmul API, computed by hand-written sm_100a kernels (libitq3.so).

See DESIGN.md for the path, the boundary and the kernels; INTEGRATION.md for the C ABI.
"""

from .codec import (BLOCK_SIZES, HEADER, MAGIC, VERSION, QuantConfig, QuantizedTensor, decode_block,
                    dequantize_tensor, encode_block, quantize_tensor, read_container, write_container)
from .compute import fused_matmul, fused_matvec
from .evaluate import (AblationRow, ErrorReport, ablate_block_size, eval_container, eval_error, generate_weights,
                       report_csv, report_json, rotation_benefit)
from .errors import (BadMagicError, ContainerError, CorruptionError, DomainError, ItqError, KernelError, LengthError,
                     ShapeError, SizeMismatchError, TruncatedStreamError, UnsupportedVersionError)
from .packing import (PackedBlock, block_nbytes, decode_f16, deserialize_block, encode_f16, pack_ternary,
                      serialize_block, unpack_ternary)
from .quantizer import (DEFAULT_SCALE_COEFF, EPSILON_D, BlockStats, ScalePolicy, TernaryGrid, argmin_scale_coeff,
                        block_stats, optimal_scale, ternary_dequantize, ternary_mse, ternary_quantize,
                        uniform_quantize)
from .selfcheck import CheckResult, run_selfcheck
from .transform import (StageTrace, fwht32_warp, fwht_forward, fwht_inverse, fwht_staged, hadamard_matrix,
                        hadamard_oracle)

__version__ = "0.1.0"

__all__ = [
    "AblationRow", "ErrorReport", "ablate_block_size", "eval_container", "eval_error", "generate_weights",
    "report_csv", "report_json", "rotation_benefit",
    "BLOCK_SIZES", "HEADER", "MAGIC", "VERSION", "DEFAULT_SCALE_COEFF", "EPSILON_D",
    "BadMagicError", "ContainerError", "CorruptionError", "DomainError", "ItqError", "KernelError", "LengthError",
    "PackedBlock", "QuantConfig", "QuantizedTensor", "ScalePolicy", "ShapeError", "SizeMismatchError", "TernaryGrid",
    "TruncatedStreamError", "UnsupportedVersionError",
    "argmin_scale_coeff", "block_nbytes", "decode_block", "decode_f16", "dequantize_tensor", "deserialize_block",
    "encode_block", "encode_f16", "fused_matmul", "fused_matvec", "fwht_forward", "fwht_inverse", "pack_ternary",
    "quantize_tensor", "read_container", "serialize_block", "unpack_ternary", "write_container",
    "BlockStats", "StageTrace", "block_stats", "fwht32_warp", "fwht_staged", "hadamard_matrix", "hadamard_oracle",
    "optimal_scale", "ternary_dequantize", "ternary_mse", "ternary_quantize", "uniform_quantize",
    "CheckResult", "run_selfcheck",
]
