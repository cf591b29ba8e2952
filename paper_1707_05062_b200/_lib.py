"""ctypes binding of the C ABI in include/kohler_cuda.h (libkohler_cuda.so).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1707_05062_b200/csrc``).  There is no fallback: if the shared
object is missing, or no sm_100 device is usable, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
# KOHLER_CUDA_LIB selects another build of the same ABI, e.g. the
# bounds-checked lib/libkohler_cuda_checked.so (tests/test_gpu_checked.py)
LIB_PATH = os.environ.get("KOHLER_CUDA_LIB") or os.path.join(LIB_DIR, "libkohler_cuda.so")
CHECKED_LIB_PATH = os.path.join(LIB_DIR, "libkohler_cuda_checked.so")
DROPIN_PATH = os.path.join(LIB_DIR, "libkohler_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(LIB_DIR), os.pardir, "include", "kohler_cuda.h")

KOHLER_OK = 0
KOHLER_NO_BOUNDARY = 1
KOHLER_INVALID_ARGUMENT = 2
KOHLER_CUDA_ERROR = 3
KOHLER_OUT_OF_MEMORY = 4
LEVELS = 256

_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int)
_vp = C.c_void_p
_sz = C.c_size_t
_i = C.c_int

# name -> (restype, argtypes); every symbol include/kohler_cuda.h declares.
SIGNATURES = {
    "kohler_cuda_abi_version": (_i, []),
    "kohler_cuda_last_error": (C.c_char_p, []),
    "kohler_cuda_create": (_i, [_i, C.POINTER(_vp)]),
    "kohler_cuda_destroy": (None, [_vp]),
    "kohler_cuda_device": (_i, [_vp]),
    "kohler_cuda_curve": (_i, [_vp, _vp, _i, _i, _sz, _vp, _vp]),
    "kohler_cuda_direct_curve": (_i, [_vp, _vp, _i, _i, _sz, _vp, _vp]),
    "kohler_cuda_analyze": (_i, [_vp, _vp, _i, _i, _sz, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kohler_cuda_analyze_batch": (
        _i, [_vp, _vp, _i, _i, _i, _sz, _sz, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kohler_cuda_mean_contrast": (_i, [_vp, _vp, _vp, _i, _vp, _vp]),
    "kohler_cuda_optimal_threshold": (_i, [_vp, _vp, _vp, _i, _vp]),
    "kohler_cuda_top_k_local_maxima": (_i, [_vp, _vp, _vp, _i, _i, _vp, _vp]),
    "kohler_cuda_analyze_batch_device": (
        _i, [_vp, _vp, _i, _i, _i, _sz, _sz, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kohler_cuda_band_curve_device": (_i, [_vp, _vp, _i, _sz, _i, _i, _i, _vp, _vp, _vp]),
    "kohler_cuda_select_device": (
        _i, [_vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kohler_cuda_last_launch_count": (_i, [_vp]),
    "kohler_cuda_set_pipeline_depth": (_i, [_vp, _i]),
    "kohler_cuda_rgb_to_gray": (_i, [_vp, _vp, _i, _i, _sz, _vp, _sz]),
    "kohler_cuda_submit": (_i, [_vp, _vp, _i, _i, _i, _sz, _sz, _i, _vp]),
    "kohler_cuda_collect": (_i, [_vp, C.c_longlong, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kohler_cuda_rgb_to_gray_device": (_i, [_vp, _vp, _i, _i, _i, _sz, _sz, _vp, _sz, _sz, _vp]),
    "kohler_cuda_analyze_rgb_batch": (
        _i, [_vp, _vp, _i, _i, _i, _sz, _sz, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kohler_cuda_analyze_rgb_batch_device": (
        _i, [_vp, _vp, _i, _i, _i, _sz, _sz, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kohler_cuda_classify": (_i, [_vp, _vp, _i, _i, _sz, _vp, _i, _vp]),
    "kohler_cuda_quantize": (_i, [_vp, _vp, _i, _i, _sz, _vp, _i, _vp]),
    "kohler_cuda_segment_batch_device": (
        _i, [_vp, _vp, _i, _i, _i, _sz, _sz, _i, _vp, _sz, _sz, _vp, _vp, _vp, _vp]),
    "kohler_cuda_segment_batch": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "kohler_cuda_multi_create": (_i, [_vp, _i, C.POINTER(_vp)]),
    "kohler_cuda_multi_destroy": (None, [_vp]),
    "kohler_cuda_multi_size": (_i, [_vp]),
    "kohler_cuda_multi_uses_nccl": (_i, [_vp]),
    "kohler_cuda_multi_uses_peer": (_i, [_vp]),
    "kohler_cuda_multi_curve": (_i, [_vp, _vp, _i, _i, _sz, _vp, _vp]),
    "kohler_cuda_multi_analyze": (
        _i, [_vp, _vp, _i, _i, _sz, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kohler_cuda_multi_analyze_batch": (
        _i, [_vp, _vp, _i, _i, _i, _sz, _sz, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


class KohlerLibraryError(RuntimeError):
    """The CUDA library is missing or failed to load (no CPU fallback exists)."""


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libkohler_cuda.so and bind every exported entry point."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise KohlerLibraryError(
                f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    return load().kohler_cuda_last_error().decode("utf-8", "replace")
