"""ctypes binding of ``libddnm.so`` (the C ABI declared in ``include/ddnm.h``).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no CPU fallback: if the
library or a CUDA device is missing, every entry point raises
:class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libddnm.so")

ABI_VERSION = 2
MAP_AUTOENCODER, MAP_LINEAR = 0, 1
ACT_SWISH, ACT_SIGMOID = 0, 1
CON_WFPC, CON_SRPC = 0, 1
STATUS_OK, STATUS_LINE_SEARCH, STATUS_KKT_SINGULAR, STATUS_LSTSQ_RANK = 0, 1, 2, 3

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


class NativeUnavailable(RuntimeError):
    """libddnm.so is missing, failed to load, or has no usable B200."""


class NativeError(RuntimeError):
    pass


class Decoder(C.Structure):
    _fields_ = [("n_out", C.c_int32), ("n_hidden", C.c_int32), ("W1", _dp), ("b1", _dp),
                ("indptr", _lp), ("indices", _lp), ("data", _dp), ("scale", _dp),
                ("shift", _dp)]


class Block(C.Structure):
    _fields_ = [("n_int", C.c_int32), ("n_gam", C.c_int32), ("interior", Decoder),
                ("interface", Decoder), ("n_rows", C.c_int32), ("res_rows", _lp),
                ("n_cols", C.c_int32), ("cols", _lp), ("n_io", C.c_int32),
                ("n_gio", C.c_int32), ("gio", _lp), ("CA", _dp), ("n_basis", C.c_int32),
                ("weights", _dp)]


class Rbf(C.Structure):
    _fields_ = [("n_centers", C.c_int32), ("n_mono", C.c_int32), ("y", _dp), ("coeffs", _dp),
                ("powers", _lp), ("shift", C.c_double * 2), ("scale", C.c_double * 2),
                ("lo", C.c_double * 2), ("hi", C.c_double * 2), ("epsilon", C.c_double)]


class Artifacts(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("map_kind", C.c_int32),
                ("activation", C.c_int32), ("gam_activation", C.c_int32),
                ("constraint_mode", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32),
                ("nu", C.c_double), ("n_blocks", C.c_int32), ("n_c", C.c_int32),
                ("blocks", C.POINTER(Block)), ("rbf", Rbf)]


class SqpCfg(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int32), ("armijo_c1", C.c_double),
                ("backtrack_factor", C.c_double), ("max_halvings", C.c_int32),
                ("reg_scale", C.c_double)]


class Info(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "n_primal", "n_mult", "n_blocks", "total_rows", "total_out_rows", "total_out_R",
        "total_int_out", "total_gam_out",
        "total_R", "total_cjac", "total_int_J", "total_gam_J", "slots_per_cta", "ctas",
        "smem_bytes", "device", "eval_units", "wide")]


class SolveOut(C.Structure):
    _fields_ = [("x", _dp), ("lam", _dp), ("n_iter", _ip), ("n_evals", _ip),
                ("status", _ip), ("n_reg", _ip), ("merit", _dp), ("objective", _dp),
                ("merit_hist", _dp), ("obj_hist", _dp), ("alpha_hist", _dp),
                ("x0", _dp), ("lam0", _dp)]


class EvalOut(C.Structure):
    _fields_ = [("rho", _dp), ("con", _dp), ("merit", _dp), ("objective", _dp), ("Br", _dp),
                ("R", _dp), ("cval", _dp), ("cjac", _dp), ("int_g", _dp), ("int_J", _dp),
                ("gam_g", _dp), ("gam_J", _dp), ("bvals", _dp), ("step", _dp),
                ("kkt_status", _ip)]


_lib = None


def lib():
    """Load libddnm.so once; raise NativeUnavailable (no fallback) on failure."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} not built; run __graft_entry__.build() (nvcc, sm_100a)")
    try:
        L = C.CDLL(LIB_PATH)
    except OSError as exc:
        raise NativeUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
    L.ddnm_last_error.restype = C.c_char_p
    L.ddnm_abi_version.restype = C.c_int
    L.ddnm_ctx_create.argtypes = [C.c_int32, C.POINTER(Artifacts), C.c_int32,
                                  C.POINTER(C.c_void_p)]
    L.ddnm_ctx_destroy.argtypes = [C.c_void_p]
    L.ddnm_ctx_info.argtypes = [C.c_void_p, C.POINTER(Info)]
    L.ddnm_solve_batch.argtypes = [C.c_void_p, C.c_int32, _dp, _dp, _dp,
                                   C.POINTER(SqpCfg), C.POINTER(SolveOut)]
    L.ddnm_solve_batch_device.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.POINTER(SqpCfg),
                                          C.POINTER(SolveOut), C.c_void_p]
    L.ddnm_eval_batch.argtypes = [C.c_void_p, C.c_int32, _dp, _dp, _dp, C.c_double,
                                  C.POINTER(EvalOut)]
    L.ddnm_last_counters.argtypes = [C.c_void_p, _lp, _lp]
    L.ddnm_last_profile.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
    L.ddnm_ctx_set_full_decoders.argtypes = [C.c_void_p, C.POINTER(Decoder),
                                             C.POINTER(Decoder)]
    L.ddnm_ctx_state_len.argtypes = [C.c_void_p, _lp]
    L.ddnm_decode_batch.argtypes = [C.c_void_p, C.c_int32, _dp, _dp, _dp, _dp]
    L.ddnm_decode_batch_device.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p]
    L.ddnm_dd_packet_len.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _lp]
    L.ddnm_dd_begin.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.POINTER(SqpCfg), C.c_int32, C.c_int32, C.POINTER(SolveOut),
                                C.c_void_p, C.POINTER(C.c_void_p), _ip]
    L.ddnm_dd_eval.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    L.ddnm_dd_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, _ip, C.c_int64, C.c_void_p,
                               _ip]
    L.ddnm_dd_end.argtypes = [C.c_void_p]
    L.ddnm_dd_set_wide.argtypes = [C.c_void_p, C.c_int32]
    L.ddnm_ctx_set_engine.argtypes = [C.c_void_p, C.c_int32]
    L.ddnm_last_rounds.argtypes = [C.c_void_p, _lp, _lp]
    L.ddnm_last_lanes.argtypes = [C.c_void_p, _lp]
    L.ddnm_wide_plan.argtypes = [C.POINTER(Artifacts), _ip, _ip]
    L.ddnm_plan_units.argtypes = [C.POINTER(Artifacts), _ip, _ip, _ip]
    L.ddnm_dd_trial_len.argtypes = [C.c_void_p, _lp]
    L.ddnm_dd_set_trials.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                     C.c_void_p]
    L.ddnm_dd_eval_p2p.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.c_int32, C.c_int32,
                                   C.c_int64, C.c_void_p]
    L.ddnm_ipc_get_handle.argtypes = [C.c_void_p, C.c_char_p]
    L.ddnm_ipc_open_handle.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    L.ddnm_ipc_close_handle.argtypes = [C.c_void_p]
    L.ddnm_dev_alloc.argtypes = [C.c_int32, C.c_int64, C.POINTER(C.c_void_p)]
    L.ddnm_dev_free.argtypes = [C.c_void_p]
    L.ddnm_binio_read.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    L.ddnm_binio_count.argtypes = [C.c_void_p, _lp]
    L.ddnm_binio_entry.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p), _lp, _lp,
                                   _lp, C.POINTER(_dp)]
    L.ddnm_binio_find.argtypes = [C.c_void_p, C.c_char_p, _lp, _lp, C.POINTER(_dp)]
    L.ddnm_binio_free.argtypes = [C.c_void_p]
    L.ddnm_binio_write.argtypes = [C.c_char_p, C.c_int64, C.POINTER(C.c_char_p), _lp, _lp,
                                   _lp, C.POINTER(_dp)]
    L.ddnm_ctx_create_binio.argtypes = [C.c_int32, C.c_char_p, C.c_int32,
                                        C.POINTER(C.c_void_p)]
    if L.ddnm_abi_version() != ABI_VERSION:
        raise NativeUnavailable("libddnm.so ABI version mismatch; rebuild")
    _lib = L
    return L


EXPORTED = ("ddnm_last_error", "ddnm_abi_version", "ddnm_ctx_create", "ddnm_ctx_destroy",
            "ddnm_ctx_info", "ddnm_solve_batch", "ddnm_solve_batch_device",
            "ddnm_eval_batch", "ddnm_last_counters", "ddnm_last_profile",
            "ddnm_ctx_set_full_decoders", "ddnm_ctx_state_len", "ddnm_decode_batch",
            "ddnm_decode_batch_device", "ddnm_dd_packet_len", "ddnm_dd_begin",
            "ddnm_dd_eval", "ddnm_dd_step", "ddnm_dd_end", "ddnm_binio_read",
            "ddnm_binio_count", "ddnm_binio_entry", "ddnm_binio_find", "ddnm_binio_free",
            "ddnm_binio_write", "ddnm_ctx_create_binio", "ddnm_dd_eval_p2p",
            "ddnm_ipc_get_handle", "ddnm_ipc_open_handle", "ddnm_ipc_close_handle",
            "ddnm_dev_alloc", "ddnm_dev_free", "ddnm_dd_trial_len", "ddnm_dd_set_trials",
            "ddnm_dd_set_wide", "ddnm_ctx_set_engine", "ddnm_last_rounds", "ddnm_last_lanes", "ddnm_wide_plan",
            "ddnm_plan_units")


def check(rc: int):
    if rc != 0:
        msg = lib().ddnm_last_error().decode(errors="replace")
        if rc == -3:
            raise NotImplementedError(msg)
        if rc == -1:
            raise ValueError(msg)
        if rc == -5:
            from .errors import FormatError
            raise FormatError(msg)
        raise NativeError(f"libddnm error {rc}: {msg}")


def ptr(a, ctype=C.c_double):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)
