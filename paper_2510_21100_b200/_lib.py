"""ctypes loader for the in-tree C-ABI library ``libhistretinex.so`` (include/histretinex.h).

Argument marshalling only.  There is no CPU fallback: if the library is missing or cannot
be loaded this module raises, and every call requires CUDA tensors.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HR_LIB selects another build of the same library (e.g. the checked build in tools/)
LIB_PATH = os.environ.get("HR_LIB") or os.path.join(HERE, "libhistretinex.so")

HR_OK, HR_EINVAL, HR_EEMPTY, HR_EDEGENERATE, HR_ECUDA, HR_EUNSUPPORTED = range(6)

# Every symbol include/histretinex.h declares (tests check the .so exports all of them).
EXPORTS = (
    "hr_default_params", "hr_create", "hr_destroy", "hr_status_string", "hr_last_error",
    "hr_version", "hr_workspace_bytes", "hr_histogram", "hr_solve", "hr_match", "hr_apply",
    "hr_enhance", "hr_enhance_debug", "hr_profile_enable", "hr_profile_collect", "hr_set_policy",
    "hr_kernel_launches", "hr_enhance_host", "hr_last_path", "hr_solve_trace", "hr_he",
    "hr_quality_workspace_bytes", "hr_quality", "hr_get_policy", "hr_trace_bind",
)


class HrDebugOut(ctypes.Structure):
    """Mirror of ``hr_debug_out`` (include/histretinex.h): nullable device pointers."""

    _fields_ = [(n, ctypes.c_void_p) for n in ("hist_s", "hist_g", "lut", "iters", "hL", "hR", "target")]


class HrParams(ctypes.Structure):
    """Mirror of ``hr_params`` (include/histretinex.h)."""

    _fields_ = [
        ("levels", ctypes.c_int32),
        ("max_iter", ctypes.c_int32),
        ("alpha", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("gamma", ctypes.c_double),
        ("epsilon", ctypes.c_double),
        ("use_epsilon", ctypes.c_int32),
        ("update_form", ctypes.c_int32),
        ("grad_norm", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class HrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


_lib = None


def load() -> ctypes.CDLL:
    """Load libhistretinex.so (raises ImportError when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    P = ctypes.POINTER(HrParams)
    sig = {
        "hr_default_params": ([P], i32),
        "hr_create": ([ctypes.POINTER(vp), ctypes.c_int], i32),
        "hr_destroy": ([vp], i32),
        "hr_status_string": ([i32], ctypes.c_char_p),
        "hr_last_error": ([vp], ctypes.c_char_p),
        "hr_version": ([], ctypes.c_char_p),
        "hr_workspace_bytes": ([i64, i32, i32], sz),
        "hr_histogram": ([vp, vp, i64, i32, i32, i32, vp, vp, vp, vp, vp], i32),
        "hr_solve": ([vp, vp, vp, i64, P, vp, vp, vp, vp, vp, vp], i32),
        "hr_solve_trace": ([vp, vp, vp, i64, P, vp, vp, vp, vp, vp, i32, vp, vp], i32),
        "hr_match": ([vp, vp, vp, i64, vp, vp, vp], i32),
        "hr_apply": ([vp, vp, vp, i64, i32, i32, vp, vp], i32),
        "hr_enhance": ([vp, vp, i64, i32, i32, P, vp, vp, vp], i32),
        "hr_enhance_debug": ([vp, vp, i64, i32, i32, P, vp, vp, ctypes.POINTER(HrDebugOut), vp], i32),
        "hr_enhance_host": ([vp, vp, i64, i32, i32, P, vp, vp, vp, vp, i32, vp], i32),
        "hr_profile_enable": ([vp, i32], i32),
        "hr_profile_collect": ([vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32)], i32),
        "hr_set_policy": ([vp, ctypes.c_char_p, i64], i32),
        "hr_get_policy": ([vp, ctypes.c_char_p, ctypes.POINTER(i64)], i32),
        "hr_kernel_launches": ([vp], i64),
        "hr_last_path": ([vp], i32),
        "hr_he": ([vp, vp, i64, i32, i32, vp, vp, vp, vp], i32),
        "hr_quality_workspace_bytes": ([i64, i32, i32], sz),
        "hr_quality": ([vp, vp, vp, i64, i32, i32, vp, vp, vp, vp, vp], i32),
        "hr_trace_bind": ([vp, vp, vp, ctypes.c_uint32], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib
