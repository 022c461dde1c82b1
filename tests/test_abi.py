"""CPU-side checks of the C ABI: libitq3.so loads, exports every symbol include/itq3.h
declares, the ctypes signatures cover them, and the host-side binary16 codec is exact."""

import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "itq3.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(itq3_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2603_27914_b200 import _lib

    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.SIGNATURES), "ctypes signature table out of sync with include/itq3.h"
    assert b"sm_100a" in lib.itq3_version()


def test_f16_codec_exhaustive_matches_numpy():
    # packing.py:87-109 semantics: every pattern round-trips; NaN canonicalises to 0x7E00
    from paper_2603_27914_b200 import decode_f16, encode_f16

    bits = np.arange(65536, dtype=np.uint16)
    vals = bits.view(np.float16).astype(np.float64)
    for b, v in zip(bits[::7], vals[::7]):
        got = decode_f16(int(b))
        assert (math.isnan(got) and math.isnan(v)) or got == v
        assert encode_f16(v) == (0x7E00 if math.isnan(v) else int(b))
    # rounding: RNE single rounding from binary64 and saturation (test_packing.py:95-105)
    assert encode_f16(2049.0) == 0x6800 and encode_f16(2051.0) == 0x6802
    assert encode_f16(1e6) == 0x7BFF and encode_f16(-1e6) == 0xFBFF
    assert encode_f16(1 + 2**-11 + 2**-40) == 0x3C01
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(2000) * 10.0 ** rng.uniform(-9, 5, 2000), [6.1e-5, 5.96e-8, 3e-8]])
    for v in x:
        with np.errstate(over="ignore"):
            want = int(np.float16(v).view(np.uint16))
        if abs(v) >= 65504:
            want = 0x7BFF | (0x8000 if v < 0 else 0)
        assert encode_f16(v) == want, v


def test_api_surface_mirrors_reference_names():
    import paper_2603_27914_b200 as P

    for name in ["QuantConfig", "QuantizedTensor", "PackedBlock", "ScalePolicy", "TernaryGrid", "quantize_tensor",
                 "dequantize_tensor", "encode_block", "decode_block", "fused_matvec", "fused_matmul",
                 "pack_ternary", "unpack_ternary", "serialize_block", "deserialize_block", "write_container",
                 "read_container", "encode_f16", "decode_f16", "fwht_forward", "fwht_inverse", "ItqError",
                 "LengthError", "DomainError", "ShapeError", "CorruptionError", "ContainerError", "BadMagicError",
                 "UnsupportedVersionError", "TruncatedStreamError", "SizeMismatchError", "BlockStats", "block_stats",
                 "optimal_scale", "ternary_quantize", "ternary_dequantize", "ternary_mse", "uniform_quantize",
                 "hadamard_matrix", "hadamard_oracle", "StageTrace", "fwht_staged", "fwht32_warp", "CheckResult",
                 "run_selfcheck", "AblationRow", "ErrorReport", "eval_error", "eval_container", "rotation_benefit",
                 "ablate_block_size", "generate_weights", "report_json", "report_csv", "argmin_scale_coeff"]:
        assert hasattr(P, name), name
    assert P.CorruptionError.ident == "corrupt-data" and issubclass(P.CorruptionError, ValueError)
    assert issubclass(P.BadMagicError, P.ContainerError) and P.SizeMismatchError.ident == "size-mismatch"


def test_no_cpu_fallback_without_gpu():
    import torch

    import paper_2603_27914_b200 as P

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.ItqError, match="no CPU fallback"):
        P.quantize_tensor(np.ones((2, 256)))


def test_host_side_layout_functions():
    """Host-only entry points (no GPU): record sizes by format flag, chain descriptor flag checks."""
    import ctypes

    from paper_2603_27914_b200 import _lib

    lib = _lib.load()
    plain = lib.itq3_mmq_nbytes(1000, 4096, 0)
    per32 = lib.itq3_mmq_nbytes(1000, 4096, 2)
    assert plain == (1024 // 128) * (4096 // 128) * (4096 + 256 + 128)
    assert per32 == (1024 // 128) * (4096 // 128) * (4096 + 1024 + 512)
    assert lib.itq3_glue_attention_ws_nbytes(32) == 32 * (16 * 130 * 4 + 4) + 4  # 16 splits + error word
    host = ctypes.create_string_buffer(lib.itq3_chain_desc_nbytes() * 2)
    # RMSNorm-input stages need the whole input in one CTA chunk (cols <= 4096)
    assert lib.itq3_chain_write_desc(host, 0, None, None, None, 1024, 4096, 4, 0) == 0
    assert lib.itq3_chain_write_desc(host, 0, None, None, None, 1024, 8192, 4, 0) != 0
    assert lib.itq3_chain_write_desc(host, 1, None, None, None, 4096, 14336, 2 | 8, 0) == 0
