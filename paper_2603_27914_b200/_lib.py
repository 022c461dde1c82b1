"""ctypes binding to libitq3.so (include/itq3.h) -- the only way into the kernels.

There is deliberately no CPU fallback: if the shared library is missing, or no CUDA
device is visible, every compute entry point raises.  PyTorch is used for device
memory and streams only (plumbing); tensors cross the ABI as raw pointers.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .errors import ItqError, from_status

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ITQ3_LIB") or os.path.join(_HERE, "lib", "libitq3.so")  # ITQ3_LIB: experiment builds

F32, F64, BF16, F16 = 0, 1, 2, 3
TORCH_DTYPE_CODE = {torch.float32: F32, torch.float64: F64, torch.bfloat16: BF16, torch.float16: F16}

CHECK_PLANES, CHECK_SCALE_NAN, CHECK_ZP, CHECK_SUB_NAN, CHECK_ZP_FINITE = 1, 2, 4, 8, 16

_i64, _i32, _u32, _vp, _dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_double

# name -> (restype, argtypes); kept in sync with include/itq3.h (tests/test_abi.py checks)
SIGNATURES = {
    "itq3_version": (ctypes.c_char_p, []),
    "itq3_last_error": (ctypes.c_char_p, []),
    "itq3_sm_count": (_i32, []),
    "itq3_copy_f32": (_i32, [_vp, _vp, _i64, _vp]),
    "itq3_encode": (_i32, [_vp, _i32, _i64, _i32, _i32, _i32, _dbl, _i32, _vp, _vp]),
    "itq3_validate": (_i32, [_vp, _i64, _i32, _i32, _u32, _vp, _vp]),
    "itq3_dequant": (_i32, [_vp, _i64, _i32, _i32, _i64, _vp, _i32, _vp]),
    "itq3_block_stats": (_i32, [_vp, _i64, _vp, _vp]),
    "itq3_ternary_quantize": (_i32, [_vp, _i64, _dbl, _i32, _vp, _vp]),
    "itq3_ternary_dequantize": (_i32, [_vp, _i64, _dbl, _i32, _vp, _vp]),
    "itq3_uniform_quantize": (_i32, [_vp, _i64, _dbl, _dbl, _dbl, _vp, _vp]),
    "itq3_glue_attention_ws_nbytes": (_i64, [_i32]),
    "itq3_glue_rope_attention": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "itq3_fwht": (_i32, [_vp, _vp, _i32, _i64, _i32, _i32, _vp]),
    "itq3_eval_ws_nbytes": (ctypes.c_size_t, [_i64, _i32]),
    "itq3_eval_ws_offset": (_i64, [_i64, _i32, _i32]),
    "itq3_eval": (_i32, [_vp, _i32, _i64, _i32, _i32, _i32, _dbl, _i32, _vp, _vp, _vp, _vp]),
    "itq3_tiled_nbytes": (_i64, [_i64, _i64, _i32]),
    "itq3_repack_tiled": (_i32, [_vp, _i64, _i64, _i32, _vp, _vp]),
    "itq3_act_nbytes": (_i64, [_i64, _i64, _i32]),
    "itq3_rotate_act": (_i32, [_vp, _i32, _i64, _i64, _i64, _i64, _i32, _vp, _vp]),
    "itq3_gemv": (_i32, [_vp, _i64, _i64, _i32, _vp, _i64, _i32, _vp, _i32, _i64, _i64, _vp]),
    "itq3_generic_ws_nbytes": (_i64, [_i64, _i64, _i32, _i64]),
    "itq3_matmul_generic": (_i32, [_vp, _i64, _i64, _i32, _i32, _vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "itq3_mmq_nbytes": (_i64, [_i64, _i64, _i32]),
    "itq3_repack_mmq": (_i32, [_vp, _i64, _i64, _i32, _vp, _vp]),
    "itq3_repack_mmq_n": (_i32, [_vp, _i64, _i64, _i32, _i32, _i32, _vp, _vp]),
    "itq3_rotate_act_f16_n": (_i32, [_vp, _i32, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _vp]),
    "itq3_mmq_block_n": (_i32, [_i64]),
    "itq3_mmq_act_nbytes": (_i64, [_i64, _i64]),
    "itq3_rotate_act_f16": (_i32, [_vp, _i32, _i64, _i64, _i64, _i64, _vp, _vp, _vp]),
    "itq3_mmq_ws_nbytes": (_i64, [_i64, _i64, _i64]),
    "itq3_mmq_set_trace": (_i32, [_vp]),
    "itq3_dequant_set_trace": (_i32, [_vp]),
    "itq3_mmq": (_i32, [_vp, _i64, _i64, _i32, _vp, _i64, _vp, _i32, _i64, _i64, _vp, _vp]),
    "itq3_mmq_peers": (_i32, [_vp, _i64, _i64, _i32, _vp, _i64, _vp, _i32, _i64, _i32, _i64, _i64, _vp, _vp]),
    "itq3_pack_codes": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp]),
    "itq3_unpack_codes": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp]),
    "itq3_mmq8_block_n": (_i32, [_i64]),
    "itq3_mmq8_nbytes": (_i64, [_i64, _i64]),
    "itq3_repack_mmq8": (_i32, [_vp, _i64, _i64, _i32, _vp, _vp]),
    "itq3_mmq8_act_nbytes": (_i64, [_i64, _i64]),
    "itq3_rotate_act_i8": (_i32, [_vp, _i32, _i64, _i64, _i64, _i64, _vp, _vp, _vp]),
    "itq3_mmq8_ws_nbytes": (_i64, [_i64, _i64, _i64]),
    "itq3_mmq8": (_i32, [_vp, _i64, _i64, _vp, _i64, _vp, _i32, _i64, _i64, _vp, _vp]),
    "itq3_chain_desc_nbytes": (_i64, []),
    "itq3_chain_act_block_bytes": (_i32, [_i32]),
    "itq3_chain_smem_bytes": (_i32, []),
    "itq3_chain_write_desc": (_i32, [_vp, _i32, _vp, _vp, _vp, _i64, _i64, _i32, _i32]),
    "itq3_chain_set_work": (_i32, [_vp, _i32, _vp]),
    "itq3_chain_set_xout": (_i32, [_vp, _i32, _vp]),
    "itq3_chain_set_xres": (_i32, [_vp, _i32, _vp]),
    "itq3_chain_write_desc_attn": (_i32, [_vp, _i32, _i32, _vp, _vp, _i64]),
    "itq3_chain_attn_params_nbytes": (_i32, []),
    "itq3_chain_write_desc_tp": (_i32, [_vp, _i32, _vp, _vp, _i64, _i64, _i32, _i64, _i64, _vp, _i32]),
    "itq3_chain_run": (_i32, [_vp, _i32, _vp, _i32, _vp, _vp, _i32, _vp, _vp]),
    "itq3_chain_run_gated": (_i32, [_vp, _i32, _vp, _i32, _vp, _vp, _i32, _vp, _vp]),
    "itq3_chain_run_ex": (_i32, [_vp, _i32, _vp, _i32, _vp, _vp, _i32, _vp, _vp, _i32]),
    "itq3_f16_encode": (ctypes.c_uint16, [_dbl]),
    "itq3_f16_decode": (_dbl, [ctypes.c_uint16]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libitq3.so (no GPU needed just to load it)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libitq3.so not built at {LIB_PATH}: run `make` at the repo root "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise ItqError("the ITQ3_S kernels need a CUDA device (sm_100a); there is no CPU fallback")
    load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(dev: torch.device | None = None) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def check(status: int) -> None:
    if status:
        raise from_status(status, load().itq3_last_error().decode())


def ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def first_bad_word(dev) -> torch.Tensor:
    return torch.full((1,), -1, dtype=torch.int64, device=dev)  # == UINT64_MAX bit pattern


def read_first_bad(word: torch.Tensor):
    v = int(word.item()) & 0xFFFFFFFFFFFFFFFF
    return None if v == 0xFFFFFFFFFFFFFFFF else v
