"""ctypes binding of libesom.so (the C ABI in include/esom.h).

This is the stub a maintainer of the reference would add:
plain pointers, sizes and a cudaStream_t, no torch types in the ABI.  The
library is built in-tree (paper_2201_00701_b200/build.py) and there is NO
fallback: if it is missing or no CUDA device is visible, every compute call
raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from .core import InputError, ParameterError

LIB_PATH = Path(__file__).resolve().parent / "libesom.so"
ESOM_OK, ESOM_ERR_PARAM, ESOM_ERR_INPUT, ESOM_ERR_CUDA, ESOM_ERR_UNSUPPORTED = range(5)

_lock = threading.Lock()
_lib = None

_vp, _i32, _i64, _f64, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_size_t

# name -> argtypes (all return int except the helpers listed below)
SIGNATURES = {
    "esom_knn": [_vp, _i64, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp],
    "esom_scores": [_vp, _i64, _i32, _vp, _vp],
    "esom_project": [_vp, _i64, _i32, _vp, _vp, _i32, _vp, _vp, _i32, _vp, _vp],
    "esom_prepare_model": [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _sz, _vp, _vp],
    "esom_embed_prepared": [_vp, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _vp, _sz, _vp, _vp, _vp, _vp, _i32, _vp,
                            _vp, _vp],
    "esom_embed_prepared_ex": [_vp, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _vp, _sz, _vp, _vp, _vp, _vp, _i32,
                               _vp, _vp, _i32, _vp, _vp],
    "esom_embed": [_vp, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _sz, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp],
    "esom_bmu_accumulate": [_vp, _i64, _i32, _vp, _i32, _vp, _sz, _vp, _vp, _vp, _i32, _vp, _vp, _vp],
    "esom_som_tick": [_vp, _i32, _vp, _i32, _vp, _vp, _i32, _f64, _f64, _vp, _sz, _vp],
    "esom_kmeans_tick": [_vp, _i32, _vp, _i32, _vp, _i32, _f64, _vp, _sz, _vp],
    "esom_batch_som_update": [_vp, _vp, _i32, _vp, _i32, _i32, _f64, _f64, _i32, _vp, _vp],
    "esom_host_register": [_vp, _sz],
    "esom_host_unregister": [_vp],
    "esom_color_channel": [_vp, _i64, _i32, _i32, _f64, _f64, _vp, _vp],
    "esom_frame_points_pack": [_vp, _vp, _i64, C.c_uint32, _vp, _vp],
    "esom_fcs_decode": [_vp, _i64, _i32, _vp, _vp, _vp],
    "esom_dim_stats": [_vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _vp],
    "esom_apply_transform": [_vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "esom_layout_tick": [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _f64, _f64, _f64, _f64, _f64, _vp, _vp, _vp, _vp],
    "esom_fit_hi": [_vp, _vp, _i32, _i32, _f64, _f64, _f64, _vp, _vp],
}
HELPERS = {
    "esom_version": ([], C.c_int),
    "esom_last_error": ([], C.c_char_p),
    "esom_workspace_bytes": ([_i32, _i32, _i32, _i32], C.c_size_t),
    "esom_tick_workspace_bytes": ([_i32, _i32], C.c_size_t),
    "esom_point_workspace_bytes": ([_i64, _i32, _i32], C.c_size_t),
    "esom_embed_workspace_bytes": ([_i64, _i32, _i32, _i32], C.c_size_t),
    "esom_embed_launches": ([_i64, _i32, _i32, _i32], C.c_int32),
    "esom_set_tc_stats": ([_vp], None),
    "esom_timing_begin": ([_i32], None),
    "esom_launch_count": ([], C.c_int64),
    "esom_timing_query": ([C.c_char_p, _vp], C.c_double),
    "esom_frame_points_bytes": ([_i64], C.c_size_t),
    "esom_mapped_device_ptr": ([_vp], _vp),
    "esom_dim_stats_workspace_bytes": ([_i64, _i32], C.c_size_t),
}


def load():
    """Load libesom.so (raises if it was not built -- no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2201_00701_b200.build` "
                "(there is no CPU fallback for the EmbedSOM kernels)")
        lib = C.CDLL(str(LIB_PATH))
        for name, argt in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argt
            fn.restype = C.c_int
        for name, (argt, rt) in HELPERS.items():
            fn = getattr(lib, name)
            fn.argtypes = argt
            fn.restype = rt
        _lib = lib
        return lib


def check(code: int) -> None:
    """Map an ESOM_ERR_* return code to the reference's exception classes."""
    if code == ESOM_OK:
        return
    msg = (load().esom_last_error() or b"").decode(errors="replace")
    if code == ESOM_ERR_PARAM:
        raise ParameterError(msg)
    if code == ESOM_ERR_INPUT:
        raise InputError(msg)
    if code == ESOM_ERR_UNSUPPORTED:
        raise UnsupportedShape(msg)
    raise RuntimeError(f"libesom error {code}: {msg}")


class UnsupportedShape(RuntimeError):
    """A kernel's shared-memory / register plan does not cover this shape
    (ESOM_ERR_UNSUPPORTED); callers with a general fallback catch it."""


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
