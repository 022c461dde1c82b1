"""B200-native ITQ3_S hot path: drop-in for the reference ``itq3`` quantize / pack /
dequantize / fused-matmul API, computed by hand-written sm_100a kernels (libitq3.so).

See DESIGN.md for the path, the boundary and the kernels; INTEGRATION.md for the C ABI.
"""

import importlib as _importlib

# Public names by defining module (the reference package's exports plus the container constants).
_EXPORTS = {
    "codec": "BLOCK_SIZES HEADER MAGIC VERSION QuantConfig QuantizedTensor decode_block dequantize_tensor "
             "encode_block quantize_tensor read_container write_container",
    "compute": "fused_matmul fused_matvec",
    "evaluate": "AblationRow ErrorReport ablate_block_size eval_container eval_error generate_weights report_csv "
                "report_json rotation_benefit",
    "errors": "BadMagicError ContainerError CorruptionError DomainError ItqError KernelError LengthError ShapeError "
              "SizeMismatchError TruncatedStreamError UnsupportedVersionError",
    "packing": "PackedBlock block_nbytes decode_f16 deserialize_block encode_f16 pack_ternary serialize_block "
               "unpack_ternary",
    "quantizer": "DEFAULT_SCALE_COEFF EPSILON_D BlockStats ScalePolicy TernaryGrid argmin_scale_coeff block_stats "
                 "optimal_scale ternary_dequantize ternary_mse ternary_quantize uniform_quantize",
    "selfcheck": "CheckResult run_selfcheck",
    "transform": "StageTrace fwht32_warp fwht_forward fwht_inverse fwht_staged hadamard_matrix hadamard_oracle",
}
for _module, _names in _EXPORTS.items():
    _m = _importlib.import_module(f"{__name__}.{_module}")
    for _name in _names.split():
        globals()[_name] = getattr(_m, _name)

__version__ = "0.1.0"
__all__ = sorted(n for names in _EXPORTS.values() for n in names.split())
del _module, _names, _m, _name
