"""ctypes binding of libcountdown_b200.so (the C-ABI in include/countdown_b200.h).

The shared library is built in-tree (``make -C paper_2505_17701_b200``, or
``__graft_entry__.build()``).  There is no fallback: if the library is missing, or a
call fails on the device, the error propagates as DataError / NumericError /
CudaError -- the same taxonomy the reference uses (errors.hpp:1-17).
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, os.environ.get("CD_LIB_DIR", "_lib"), "libcountdown_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "countdown_b200.h")

CD_OK, CD_ERR_USAGE, CD_ERR_DATA, CD_ERR_NUMERIC, CD_ERR_CUDA = 0, 1, 2, 3, 4
ACT_SILU, ACT_GELU_TANH = 0, 1
DTYPE_F32, DTYPE_BF16 = 0, 1
REDUCTION_ORDERED, REDUCTION_UNORDERED = 0, 1
METHOD_DENSE, METHOD_MC, METHOD_DC, METHOD_CATS = 0, 1, 2, 3
ENGINE_FUSED, ENGINE_TENSOR, ENGINE_HOST_GRAPH, ENGINE_ALL, ENGINE_PDL_CHAIN = 1, 2, 4, 7, 8


class DataError(RuntimeError):
    """countdown::DataError (errors.hpp:11-13): bad inputs, shapes or arguments."""


class NumericError(RuntimeError):
    """countdown::NumericError (errors.hpp:15-17): non-finite results."""


class CudaError(RuntimeError):
    """Device failure (no reference equivalent: the reference has no device)."""


_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int
_f32 = C.c_float
_u64 = C.c_uint64

# name -> argtypes (restype int unless listed in _RESTYPES)
_SIGNATURES = {
    "cd_last_error": [],
    "cd_version": [],
    "cd_device_info": [_i32, _vp, _vp, _vp],
    "cd_layer_create": [_i32, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _vp],
    "cd_layer_create_shard": [_i32, _i64, _i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _vp],
    "cd_layer_set_predictor": [_vp, _i64, _vp, _vp],
    "cd_layer_load_cdwn1": [_i32, C.c_char_p, _i32, _vp, _vp],
    "cd_layer_destroy": [_vp],
    "cd_layer_shape": [_vp, _vp, _vp, _vp, _vp, _vp],
    "cd_layer_device_bytes": [_vp, _vp],
    "cd_layer_last_launches": [_vp, _vp],
    "cd_layer_last_path": [_vp, _vp],
    "cd_exec_dense": [_vp, _i64, _vp, _i32, _vp],
    "cd_exec_mc": [_vp, _i64, _vp, _vp, _vp, _i32, _vp],
    "cd_exec_dc": [_vp, _i64, _vp, _vp, _i32, _vp],
    "cd_pipeline_mc": [_vp, _i64, _vp, _f32, _i32, _vp, _vp, _vp, _vp],
    "cd_exec_cats": [_vp, _i64, _vp, _vp, _vp, _i32, _vp],
    "cd_pipeline_cats": [_vp, _i64, _vp, _f32, _i32, _vp, _vp, _vp, _vp],
    "cd_pipeline_dc": [_vp, _i64, _vp, _f32, _vp, _i32, _vp, _vp, _vp, _vp],
    "cd_predict_logits": [_vp, _i64, _vp, _vp],
    "cd_forward_device": [_vp, _i32, _i64, _vp, _f32, _i32, _vp, _vp, _vp, _vp, _vp, _vp],
    "cd_forward_device_normed": [_vp, _i32, _i64, _vp, _f32, _f32, _i32, _vp, _vp, _vp, _vp, _vp, _vp],
    "cd_layer_sync": [_vp],
    "cd_layer_set_prefetch": [_vp, _vp],
    "cd_top_m": [_i32, _i64, _i64, _vp, _i64, _i32, _vp, _vp],
    "cd_top_m_device": [_vp, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _vp],
    "cd_calibrate": [_vp, _i32, _i64, _vp, C.c_double, _vp, _vp],
    "cd_layer_set_engines": [_vp, _i32],
    "cd_predictor_create": [_i32, _i64, _i64, _i64, _i32, _vp, _vp, _vp],
    "cd_predictor_create_ternary": [_i32, _i64, _i64, _f32, _vp, _vp],
    "cd_bench_device": [_vp, _i32, _i64, _vp, _f32, _i32, _i64, _i64, _vp],
    "cd_bench_stages": [_vp, _i32, _i32, _i64, _vp, _f32, _i64, _i64, _vp, _vp],
    "cd_synth_layer": [_u64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp],
    "cd_synth_normals": [_u64, _i64, _vp],
}
_RESTYPES = {"cd_last_error": C.c_char_p}

_lib = None


def header_symbols() -> list[str]:
    """Every function the public header declares (CD_API ... cd_xxx( )."""
    with open(HEADER_PATH) as f:
        text = f.read()
    return re.findall(r"CD_API\s+[\w\s\*]+?\b(cd_\w+)\s*\(", text)


def lib() -> C.CDLL:
    """Load the in-tree library (once).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaError(
                f"{LIB_PATH} is missing: build it with `make -C {HERE}` or "
                f"`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, argtypes in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == CD_OK:
        return
    msg = lib().cd_last_error().decode(errors="replace")
    if rc == CD_ERR_DATA:
        raise DataError(msg)
    if rc == CD_ERR_NUMERIC:
        raise NumericError(msg)
    if rc == CD_ERR_CUDA:
        raise CudaError(msg)
    raise RuntimeError(f"countdown_b200 error {rc}: {msg}")


def ptr(a) -> C.c_void_p | None:
    """Raw pointer of a numpy array (C-contiguous) or torch tensor; None passes NULL."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)
