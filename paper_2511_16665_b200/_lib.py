"""ctypes binding of libtlt_b200.so (the C-ABI declared in include/tlt_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()``. There is no
fallback: importing the product path without the extension raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtlt_b200.so")

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'). No CPU fallback exists.")
        _lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        _declare(_lib)
    return _lib


i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)
f32p = C.POINTER(C.c_float)


def _declare(L: C.CDLL) -> None:
    L.tlt_version.restype = C.c_char_p
    L.tlt_last_error.restype = C.c_char_p
    L.tlt_last_error.argtypes = [C.c_void_p]
    L.tlt_rng_next_u64.restype = C.c_uint64
    L.tlt_rng_next_u64.argtypes = [C.c_void_p]
    L.tlt_rng_uniform01.restype = C.c_double
    L.tlt_rng_uniform01.argtypes = [C.c_void_p]
    L.tlt_rng_destroy.argtypes = [C.c_void_p]
    L.tlt_engine_destroy.argtypes = [C.c_void_p]
    L.tlt_c1_destroy.argtypes = [C.c_void_p]
    L.tlt_mab_destroy.argtypes = [C.c_void_p]
    L.tlt_ngram_destroy.argtypes = [C.c_void_p]
    L.tlt_ngram_draft.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    L.tlt_dev_time_gemm.restype = C.c_int
    L.tlt_dev_time_gemm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_longlong, C.c_int, C.c_void_p]
    L.tlt_dev_gemm.restype = C.c_int
    L.tlt_dev_gemm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_int]
    L.tlt_dev_lm_topk.restype = C.c_int
    L.tlt_dev_lm_topk.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 6
    L.tlt_dev_gemm_live.restype = C.c_int
    L.tlt_dev_gemm_live.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p]
    L.tlt_dev_gemm_e4m3.restype = C.c_int
    L.tlt_dev_gemm_e4m3.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int] + [C.c_void_p] * 5
    L.tlt_dev_attention.restype = C.c_int
    L.tlt_dev_attention.argtypes = [C.c_void_p] * 4 + [C.c_int] * 6 + [C.c_void_p] * 6 + [C.c_int] * 2
    L.tlt_dev_row_topk.restype = C.c_int
    L.tlt_dev_row_topk.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]


def last_error(engine=None) -> str:
    msg = lib().tlt_last_error(engine)
    return msg.decode() if msg else ""


class TltError(RuntimeError):
    pass


def check(rc: int, engine=None) -> int:
    """Raise on a negative return of the kernel-level dev entry points (which
    return a count, or -1 with tlt_last_error set); pass the count through."""
    if rc < 0:
        raise TltError(last_error(engine))
    return rc
