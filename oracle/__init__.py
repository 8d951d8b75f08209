"""ctypes access to the CPU oracle (TEST INFRASTRUCTURE ONLY).

``liboracle.so``  — C restatement of the reference hot path + neural oracle.
``_ref/libspecsim_ref.so`` — extern "C" bridge over the unmodified reference
headers, compiled in place from /root/reference (travels prebuilt).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspecsim_ref.so")

i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)
ROW_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, i32p, C.c_int, f64p)
ARGMAX_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, i32p, C.c_int)


class Strategy(C.Structure):
    _fields_ = [("draft_depth", C.c_int32), ("top_k", C.c_int32), ("tokens_to_verify", C.c_int32)]


class Node(C.Structure):
    _fields_ = [("token", C.c_int32), ("parent", C.c_int32), ("depth", C.c_int32), ("prob", C.c_double),
                ("path_prob", C.c_double)]


class Accept(C.Structure):
    _fields_ = [("accepted", C.c_int32 * 256), ("nodes", C.c_int32 * 256), ("accept_length", C.c_int32),
                ("bonus", C.c_int32)]


class USrc(C.Structure):
    _fields_ = [("rng", C.c_void_p), ("buf", f64p), ("n", C.c_int), ("cursor", C.c_int)]


class Capture(C.Structure):
    _fields_ = [("side", C.c_int32), ("bucket_lo", C.c_int32), ("bucket_hi", C.c_int32),
                ("tokens_to_verify", C.c_int32), ("top_k", C.c_int32), ("draft_depth", C.c_int32),
                ("memory_units", C.c_double)]


class TestRows(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("vocab", C.c_int), ("levels", C.c_int), ("zero_pct", C.c_int)]


class ModelCfg(C.Structure):
    _fields_ = [("vocab", C.c_int), ("hidden", C.c_int), ("layers", C.c_int), ("heads", C.c_int),
                ("kv_heads", C.c_int), ("head_dim", C.c_int), ("ffn", C.c_int), ("qkv_bias", C.c_int),
                ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("max_ctx", C.c_int)]


class InitCfg(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("layer_scale", C.c_float), ("lm_gain", C.c_float), ("lm_alt", C.c_float),
                ("lm_noise", C.c_float), ("fc_noise", C.c_float),
                ("drafter_lm_fp8", C.c_int32)]


_orc = None
_ref = None


def build() -> None:
    """Build liboracle.so (and the reference bridge when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.orc_rng_sizeof.restype = C.c_size_t
        L.orc_mab_sizeof.restype = C.c_size_t
        L.orc_rng_next_u64.restype = C.c_uint64
        L.orc_rng_uniform01.restype = C.c_double
        L.orc_rng_uniform_int.restype = C.c_uint64
        L.orc_rng_uniform_int.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_normal.restype = C.c_double
        L.orc_rng_init.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.orc_rng_fork.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.orc_median.restype = C.c_double
        L.orc_step_latency.restype = C.c_double
        L.orc_max_tree_nodes.restype = C.c_int64
        L.orc_now.restype = C.c_double
        if hasattr(L, 'orc_model_create'):
            L.orc_model_create.restype = C.c_void_p
            L.orc_model_create.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
            L.orc_model_destroy.argtypes = [C.c_void_p]
            L.orc_seq_create.restype = C.c_void_p
            L.orc_seq_create.argtypes = [C.c_void_p]
            L.orc_seq_destroy.argtypes = [C.c_void_p]
            L.orc_init_value.restype = C.c_uint16
            L.orc_init_value.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int64]
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        for name in ["ref_rng_create", "ref_rng_fork", "ref_mab_create", "ref_make_random_model",
                     "ref_make_cyclic_model"]:
            getattr(L, name).restype = C.c_void_p
        L.ref_rng_create.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_rng_fork.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_rng_destroy.argtypes = [C.c_void_p]
        L.ref_rng_next_u64.restype = C.c_uint64
        L.ref_rng_next_u64.argtypes = [C.c_void_p]
        L.ref_rng_uniform01.restype = C.c_double
        L.ref_rng_uniform01.argtypes = [C.c_void_p]
        L.ref_rng_uniform_int.restype = C.c_uint64
        L.ref_rng_uniform_int.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_rng_normal.restype = C.c_double
        L.ref_rng_normal.argtypes = [C.c_void_p]
        L.ref_max_tree_nodes.restype = C.c_longlong
        L.ref_step_latency.restype = C.c_double
        L.ref_mab_create.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_void_p]
        L.ref_mab_destroy.argtypes = [C.c_void_p]
        L.ref_mab_select.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.ref_mab_record.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int,
                                     C.c_int]
        L.ref_mab_stats.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p]
        L.ref_make_random_model.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_void_p]
        L.ref_make_cyclic_model.argtypes = [C.c_int, C.c_void_p, C.c_int]
        L.ref_model_destroy.argtypes = [C.c_void_p]
        L.ref_generate_autoregressive.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_uint64,
                                                  C.c_void_p, C.c_void_p]
        L.ref_spec_generate_greedy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                               C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_void_p]
        L.ref_verify_stochastic.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_int,
                                            C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p]
        L.ref_build_sampled_chain.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_verify_greedy.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_build_draft_tree.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_plan_captures.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                        C.c_void_p, C.c_int, C.c_void_p]
        L.ref_target_next_dist.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_void_p]
        L.ref_argmax.argtypes = [C.c_void_p, C.c_int]
        L.ref_inverse_cdf_pick.argtypes = [C.c_void_p, C.c_int, C.c_double]
        L.ref_sample_response_length.argtypes = [C.c_double, C.c_double, C.c_int, C.c_void_p]
        _ref = L
    return _ref


def fnptr(lib: C.CDLL, name: str) -> C.c_void_p:
    """Raw C function pointer of an exported symbol (passed as a row callback)."""
    return C.cast(getattr(lib, name), C.c_void_p)


class Rng:
    """orc_rng wrapper (C restatement of RngStream)."""

    def __init__(self, seed: int = 0, stream: int = 0, _buf=None):
        L = orc()
        self.buf = _buf if _buf is not None else C.create_string_buffer(L.orc_rng_sizeof())
        if _buf is None:
            L.orc_rng_init(self.buf, seed, stream)

    def fork(self, label: int) -> "Rng":
        L = orc()
        out = C.create_string_buffer(L.orc_rng_sizeof())
        L.orc_rng_fork(self.buf, label, out)
        return Rng(_buf=out)

    def next_u64(self) -> int:
        return orc().orc_rng_next_u64(self.buf)

    def uniform01(self) -> float:
        return orc().orc_rng_uniform01(self.buf)

    def uniform_int(self, n: int) -> int:
        return orc().orc_rng_uniform_int(self.buf, n)

    def normal(self) -> float:
        return orc().orc_rng_normal(self.buf)
