"""ctypes binding of libgks.so (the C ABI declared in include/gks.h).

There is no fallback: if the shared library is missing or no CUDA device is
visible, calls raise.  Build with `python -m paper_2304_09485_b200.build` or
`__graft_entry__.build()`.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libgks.so"

GKS_OK = 0
GKS_ERR_BAD_ARG = 1
GKS_ERR_CUDA = 2
GKS_ERR_UNPHYSICAL = 3
GKS_ERR_SINGULAR = 4
GKS_ERR_NONFINITE = 5
GKS_ERR_MESH = 6
GKS_ERR_NCCL = 7
GKS_ERR_NO_DEVICE = 8
GKS_ERR_INVALID_UPDATE = 9

_lock = threading.Lock()
_lib = None

c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)
c_int32_p = C.POINTER(C.c_int32)
c_void_p = C.c_void_p


class GksError(RuntimeError):
    def __init__(self, code, message, index=-1):
        super().__init__(message)
        self.code = code
        self.index = index


# (name, restype, argtypes) of every exported symbol; kept in sync with
# include/gks.h (tests/test_native_abi.py checks both directions).
SIGNATURES = [
    ("gks_abi_version", C.c_int, []),
    ("gks_last_error", C.c_char_p, []),
    ("gks_last_error_index", C.c_int64, []),
    ("gks_kernel_launches", C.c_int64, []),
    ("gks_flux_batch", C.c_int, [C.c_int64, c_double_p, c_double_p, c_double_p, c_double_p,
                                 c_double_p, c_double_p, c_double_p, C.c_double, c_double_p,
                                 c_double_p]),
    ("gks_flux_bench", C.c_int, [C.c_int64, C.c_int, C.c_double, c_double_p]),
]


def load():
    """Load libgks.so once (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -m paper_2304_09485_b200.build); there is no CPU fallback")
        lib = C.CDLL(str(LIB_PATH))
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc):
    if rc != GKS_OK:
        lib = load()
        msg = lib.gks_last_error().decode(errors="replace")
        raise GksError(rc, msg, int(lib.gks_last_error_index()))


def dptr(a):
    """Pointer to a C-contiguous float64 array (None -> NULL)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(c_double_p)


def iptr(a):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(c_int64_p)


def i32ptr(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(c_int32_p)


def f64(a, shape=None):
    out = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        out = out.reshape(shape)
    return out


def kernel_launches():
    return int(load().gks_kernel_launches())
