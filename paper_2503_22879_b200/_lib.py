"""ctypes binding of libssmquant_sm100.so (include/ssmquant_sm100.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).  There is
no fallback: if the library is missing or the device is not sm_100, every op raises.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_NAME = "libssmquant_sm100.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
ABI_VERSION = 8

_i8p = C.c_void_p
_f32p = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
_flt = C.c_float
_vp = C.c_void_p


class Mamba2Params(C.Structure):
    _fields_ = [("n_heads", _int), ("head_dim", _int), ("d_state", _int), ("n_groups", _int),
                ("head_group", _vp), ("A", _vp), ("D", _vp), ("dt_bias", _vp),
                ("s_dt", _flt), ("s_z", _flt), ("s_x", _vp), ("s_B", _vp), ("s_C", _vp), ("s_h", _vp)]


class Mamba2DecodeParams(C.Structure):
    _fields_ = [("ssm", Mamba2Params), ("conv_kernel", _int), ("conv_w", _vp), ("conv_b", _vp), ("conv_s_in", _vp),
                ("conv_s_out", _vp), ("norm_w", _vp), ("eps", _flt), ("s_y", _flt), ("hadamard", _int)]


class Mamba1Params(C.Structure):
    _fields_ = [("d_inner", _int), ("d_state", _int), ("A", _vp), ("D", _vp), ("dt_bias", _vp),
                ("s_dt", _flt), ("s_z", _flt), ("s_B", _flt), ("s_C", _flt), ("s_x", _vp), ("s_h", _vp)]


class Mamba1DecodeParams(C.Structure):
    _fields_ = [("ssm", Mamba1Params), ("conv_kernel", _int), ("conv_w", _vp), ("conv_b", _vp), ("conv_s_in", _vp),
                ("conv_s_out", _vp), ("dt_rank", _int), ("xproj_w", _vp), ("xproj_alpha", _vp), ("xproj_cs", _vp),
                ("dtproj_w", _vp), ("dtproj_alpha", _vp), ("dtproj_cs", _vp), ("norm_w", _vp), ("eps", _flt),
                ("s_y", _flt), ("hadamard", _int)]


class Mamba1LayerParams(C.Structure):
    _fields_ = [("ln_w", _vp), ("ln_eps", _flt), ("s_u", _flt), ("d_model", _int), ("in_w", _vp), ("in_alpha", _vp),
                ("in_cs", _vp), ("out_w", _vp), ("out_alpha", _vp)]


class ConvEpilogue(C.Structure):
    _fields_ = [("w", _vp), ("b", _vp), ("kc", _int), ("c0", _int), ("C", _int), ("cache", _vp), ("cache_in", _int),
                ("out", _vp), ("ldo", _i64)]


_SIGS = {
    "sq_abi_version": ([], _int),
    "sq_last_error": ([], C.c_char_p),
    "sq_device_supported": ([], _int),
    "sq_w4_bytes": ([_int, _int], _i64),
    "sq_repack_w4": ([_vp, _int, _int, _vp, _vp], _int),
    "sq_unpack_w4": ([_vp, _int, _int, _vp, _vp], _int),
    "sq_rmsnorm_quant": ([_vp, _i64, _vp, _flt, _flt, _int, _int, _vp, _i64, _vp, _i64, _vp], _int),
    "sq_rmsnorm_f32": ([_vp, _i64, _vp, _flt, _int, _int, _vp, _i64, _vp], _int),
    "sq_quantize_f32": ([_vp, _i64, _flt, _int, _int, _vp, _i64, _vp], _int),
    "sq_embed_int8": ([_vp, _vp, _vp, _int, _int, _vp, _vp], _int),
    "sq_embed_u4": ([_vp, _vp, _vp, _int, _int, _vp, _vp], _int),
    "sq_argmax_f32": ([_vp, _i64, _int, _int, _vp, _vp], _int),
    "sq_gemm_w8a8": ([_vp, _i64, _vp, _vp, _int, _int, _int, _int, _vp, _i64, _vp, _vp], _int),
    "sq_gemm_w4a8": ([_vp, _i64, _vp, _vp, _int, _flt, _int, _int, _int, _int, _vp, _i64, _vp, _vp], _int),
    "sq_gemm_w4a8_splits": ([_int, _int, _int], _int),
    "sq_group_scale_elems": ([_int, _int], _i64),
    "sq_tile_group_scales": ([_vp, _int, _int, _vp, _vp], _int),
    "sq_w4a16_bytes": ([_int, _int, _int], _i64),
    "sq_repack_w4a16": ([_vp, _int, _int, _int, _vp, _vp], _int),
    "sq_gemv_w4a16": ([_vp, _i64, _vp, _flt, _vp, _vp, _int, _int, _int, _int, _vp, _i64, _int, _vp], _int),
    "sq_gemv_w4a16_conv": ([_vp, _i64, _vp, _flt, _vp, _vp, _int, _int, _int, _int, _vp, _i64, _int,
                            C.POINTER(ConvEpilogue), _vp], _int),
    "sq_conv1d_int8": ([_vp, _i64, _vp, _vp, _vp, _vp, _int, _int, _int, _int, _vp, _int, _vp, _i64, _vp], _int),
    "sq_conv1d_update_int8": ([_vp, _i64, _vp, _vp, _vp, _vp, _int, _int, _int, _vp, _vp, _i64, _vp], _int),
    "sq_conv1d_f32": ([_vp, _i64, _vp, _vp, _int, _int, _int, _int, _vp, _int, _vp, _i64, _vp], _int),
    "sq_ssd_scan_int8": ([C.POINTER(Mamba2Params), _int, _int, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _i64,
                          _vp, _int, _vp, _i64, _int, _vp], _int),
    "sq_state_update_int8": ([C.POINTER(Mamba2Params), _int, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _i64,
                              _vp, _vp, _i64, _vp], _int),
    "sq_ssd_scan_f32": ([C.POINTER(Mamba2Params), _int, _int, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _i64,
                         _vp, _int, _vp, _i64, _vp], _int),
    "sq_selective_scan_int8_ws_bytes": ([C.POINTER(Mamba1Params), _int, _int], _i64),
    "sq_selective_scan_int8": ([C.POINTER(Mamba1Params), _int, _int, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64,
                                _vp, _int, _vp, _i64, _vp, _vp], _int),
    "sq_selective_scan_f32": ([C.POINTER(Mamba1Params), _int, _int, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64,
                                _vp, _int, _vp, _i64, _vp], _int),
    "sq_mamba1_decode_ws_bytes": ([C.POINTER(Mamba1DecodeParams), _int], _i64),
    "sq_mamba1_decode_layer_int8": ([C.POINTER(Mamba1DecodeParams), C.POINTER(Mamba1LayerParams), _int, _vp, _i64,
                                     _vp, _vp, _vp, _vp], _int),
    "sq_mamba1_decode_step_int8": ([C.POINTER(Mamba1DecodeParams), _int, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp],
                                   _int),
    "sq_mamba2_decode_ws_bytes": ([C.POINTER(Mamba2DecodeParams), _int], _i64),
    "sq_mamba2_decode_launches": ([C.POINTER(Mamba2DecodeParams), _int, _int], _int),
    "sq_mamba2_decode_step_int8": ([C.POINTER(Mamba2DecodeParams), _int, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp,
                                    _i64, _vp, _i64, _vp], _int),
    "sq_gate_norm_had_quant": ([_vp, _i64, _vp, _flt, _flt, _int, _int, _int, _vp, _i64, _vp], _int),
    "sq_discretize_f32": ([_vp, _i64, _vp, _vp, _int, _int, _int, _vp, _vp, _vp], _int),
    "sq_selective_scan2_pre_f32": ([C.POINTER(Mamba2Params), _int, _int, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64,
                                    _vp, _i64, _vp, _int, _vp, _i64, _vp], _int),
    "sq_selective_scan1_pre_f32": ([C.POINTER(Mamba1Params), _int, _int, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64,
                                    _vp, _i64, _vp, _int, _vp, _i64, _vp], _int),
}

EXPORTS = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load and type the library (no device work).  Raises if it is absent."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.sq_abi_version() != ABI_VERSION:
        raise RuntimeError(f"ABI mismatch: {lib.sq_abi_version()} != {ABI_VERSION}")
    if path == LIB_PATH:
        _lib = lib
    return lib


def last_error() -> str:
    return load().sq_last_error().decode("utf-8", "replace")
