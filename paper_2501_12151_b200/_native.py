"""ctypes binding of libqtt.so (include/qtt.h).

The library is built in-tree by ``__graft_entry__.build()`` (csrc/Makefile).  There is
no CPU fallback: if the library or a CUDA device is missing, every call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import CapacityError, DeviceError, FormatError, ShapeMismatchError, SolverError

# QTT_LIB overrides the library path (A/B timing of two builds on one GPU box)
LIB_PATH = os.environ.get("QTT_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libqtt.so")

_lib = None
_lock = threading.Lock()

QTT_OK, QTT_ERR_SHAPE, QTT_ERR_SOLVER, QTT_ERR_CAPACITY, QTT_ERR_CUDA, QTT_ERR_ARG, QTT_ERR_FORMAT = range(7)

_P = ctypes.POINTER(ctypes.c_double)
_I = ctypes.c_int
_VP = ctypes.c_void_p


class QttStats(ctypes.Structure):
    _fields_ = [
        ("launches", ctypes.c_int64), ("k1_calls", ctypes.c_int64),
        ("k1_flops", ctypes.c_double), ("k1_ms", ctypes.c_double),
        ("env_calls", ctypes.c_int64), ("env_flops", ctypes.c_double), ("env_ms", ctypes.c_double),
        ("cg_iters", ctypes.c_int64), ("cg_solves", ctypes.c_int64), ("chol_solves", ctypes.c_int64),
        ("svd_calls", ctypes.c_int64), ("qr_calls", ctypes.c_int64), ("sweeps", ctypes.c_int64),
        ("certifications", ctypes.c_int64),
        ("k1_timed_flops", ctypes.c_double), ("env_timed_flops", ctypes.c_double),
        ("phase_ms", ctypes.c_double * 10),
    ]

PHASES = ("other", "direct", "cg", "mixed_res", "svd", "qr", "env", "cert", "prepass", "rhs")


# name -> argtypes (restype is int unless listed in _RESTYPES)
SIGNATURES = {
    "qtt_version": [],
    "qtt_last_error": [],
    "qtt_ctx_create": [_I, ctypes.POINTER(_VP)],
    "qtt_ctx_destroy": [_VP],
    "qtt_ctx_synchronize": [_VP],
    "qtt_ctx_stream": [_VP],
    "qtt_ctx_set_profiling": [_VP, _I],
    "qtt_ctx_get_stats": [_VP, ctypes.POINTER(QttStats)],
    "qtt_ctx_reset_stats": [_VP],
    "qtt_ctx_flush_l2": [_VP],
    "qtt_launch_count": [],
    "qtt_ctx_trace": [_VP, ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)],
    "qtt_local_matvec": [_VP, _P, _P, _P, _P] + [_I] * 8 + [_P],
    "qtt_env_left": [_VP, _P, _P, _P, _P] + [_I] * 8 + [_P],
    "qtt_env_right": [_VP, _P, _P, _P, _P] + [_I] * 8 + [_P],
    "qtt_psi_left": [_VP, _P, _P, _P] + [_I] * 5 + [_P],
    "qtt_psi_right": [_VP, _P, _P, _P] + [_I] * 5 + [_P],
    "qtt_local_rhs": [_VP, _P, _P, _P] + [_I] * 5 + [_P],
    "qtt_local_dense": [_VP, _P, _P, _P] + [_I] * 8 + [_P],
    "qtt_local_diag": [_VP, _P, _P, _P] + [_I] * 5 + [_P],
    "qtt_mixed_residual": [_VP] + [_P] * 7 + [_I] * 10 + [_P],
    "qtt_train_upload": [_VP, _I, _I, ctypes.POINTER(ctypes.c_int64), _P, ctypes.POINTER(_VP)],
    "qtt_train_info": [_VP, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(ctypes.c_int64)],
    "qtt_train_shape": [_VP, ctypes.POINTER(ctypes.c_int64)],
    "qtt_train_download": [_VP, _VP, _P],
    "qtt_train_free": [_VP],
    "qtt_train_load_qtt1": [_VP, ctypes.c_char_p, ctypes.POINTER(_I), ctypes.POINTER(_VP)],
    "qtt_train_save_qtt1": [_VP, _VP, ctypes.c_char_p],
    "qtt_orthogonalize_rl": [_VP, _VP, ctypes.POINTER(_VP)],
    "qtt_tt_norm": [_VP, _VP, _P],
    "qtt_tt_dot": [_VP, _VP, _VP, _P],
    "qtt_tt_round": [_VP, _VP, ctypes.c_double, _I, ctypes.POINTER(_VP)],
    "qtt_tt_apply": [_VP, _VP, _VP, ctypes.POINTER(_VP)],
    "qtt_tt_apply_into": [_VP, _VP, _VP, _VP],
    "qtt_tt_entries": [_VP, _VP, ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, _P],
    "qtt_tt_to_dense": [_VP, _VP, ctypes.c_int64, _P],
    "qtt_matvec_sweep": [_VP, _VP, _VP, _I, ctypes.POINTER(_VP), _P],
    "qtt_residual_norm": [_VP, _VP, _VP, _VP, _I, _P, ctypes.POINTER(_I)],
    "qtt_qr": [_VP, _P, _I, _I, _P, _P],
    "qtt_svd": [_VP, _P, _I, _I, _P, _P, _P],
    "qtt_rank_for_tolerance": [_P, _I, ctypes.c_double, ctypes.POINTER(_I)],
    "qtt_local_solve": [_VP, _P, _P, _P, _P, _P] + [_I] * 7 + [ctypes.c_double, _I, _I, _P, _P,
                                                                 ctypes.POINTER(_I)],
    "qtt_amen_solve": [_VP, _VP, _VP, _VP, ctypes.c_void_p, _P, ctypes.c_int64, ctypes.POINTER(_VP),
                       ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), _P],
    "qtt_maxvol": [_VP, _P, _I, _I, _I, ctypes.c_double, _I, ctypes.POINTER(ctypes.c_int32), _P,
                   ctypes.POINTER(_I)],
    "qtt_amen_step": [_VP, _VP, _VP, ctypes.c_void_p, _I, _I, _I, ctypes.c_double, ctypes.c_double, _I,
                      ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_VP), _P,
                      ctypes.POINTER(_I), ctypes.POINTER(_I)],
}


class AmenParams(ctypes.Structure):
    _fields_ = [
        ("residual_tol", ctypes.c_double), ("max_sweeps", ctypes.c_int),
        ("enrichment_rank", ctypes.c_int), ("local_iterative", ctypes.c_int),
        ("direct_dim_cap", ctypes.c_int), ("local_iter_cap", ctypes.c_int),
        ("round_tol", ctypes.c_double), ("round_max_rank", ctypes.c_int),
        ("stagnation_strikes", ctypes.c_int), ("fused_cg", ctypes.c_int),
    ]


class AmenReport(ctypes.Structure):
    _fields_ = [
        ("converged", ctypes.c_int), ("sweeps_used", ctypes.c_int),
        ("final_relative_residual", ctypes.c_double),
        ("certifications_gram", ctypes.c_int), ("certifications_exact", ctypes.c_int),
        ("draws_used", ctypes.c_int64),
    ]
_RESTYPES = {"qtt_last_error": ctypes.c_char_p, "qtt_ctx_stream": _VP, "qtt_launch_count": ctypes.c_int64}


def load_library(path: str = LIB_PATH):
    """Load and type the shared library (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"{path} is missing; build it with __graft_entry__.build() "
                "(the QTT engine has no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
        return lib


def check(code: int):
    if code == QTT_OK:
        return
    msg = _lib.qtt_last_error().decode(errors="replace")
    if code == QTT_ERR_SHAPE:
        raise ShapeMismatchError(msg)
    if code == QTT_ERR_SOLVER:
        raise SolverError(msg)
    if code == QTT_ERR_CAPACITY:
        raise CapacityError(msg)
    if code == QTT_ERR_FORMAT:
        raise FormatError(msg)
    if code == QTT_ERR_ARG:
        raise ValueError(msg)
    raise DeviceError(msg)


def call(name: str, *args):
    lib = load_library()
    check(getattr(lib, name)(*args))


class Context:
    """One engine context (CUDA stream + memory pool) on one device."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = _VP()
        check(lib.qtt_ctx_create(int(device), ctypes.byref(h)))
        self.handle = h
        self.device = device

    def close(self):
        if self.handle:
            _lib.qtt_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        call("qtt_ctx_synchronize", self.handle)

    @property
    def stream(self) -> int:
        return _lib.qtt_ctx_stream(self.handle)

    def set_profiling(self, on, phases: bool = False):
        """on: CUDA-event timing of K1/K2 launches; phases: synchronizing per-phase wall timing."""
        call("qtt_ctx_set_profiling", self.handle, (1 if on else 0) | (2 if phases else 0))

    def flush_l2(self):
        call("qtt_ctx_flush_l2", self.handle)

    def stats(self) -> dict:
        s = QttStats()
        call("qtt_ctx_get_stats", self.handle, ctypes.byref(s))
        out = {name: getattr(s, name) for name, _ in QttStats._fields_ if name != "phase_ms"}
        out["phase_ms"] = {PHASES[i]: float(s.phase_ms[i]) for i in range(10)}
        return out

    def reset_stats(self):
        call("qtt_ctx_reset_stats", self.handle)

    TRACE_FIELDS = ("sweep", "core", "rl", "m", "rr", "zl", "zr", "R0", "R1", "path", "iters")

    def trace(self) -> np.ndarray:
        """(n, 11) int32 array of local-solve records since the last reset_stats()."""
        n = ctypes.c_int64()
        call("qtt_ctx_trace", self.handle, None, 0, ctypes.byref(n))
        out = np.zeros((max(n.value, 1), 11), dtype=np.int32)
        call("qtt_ctx_trace", self.handle, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
             n.value, ctypes.byref(n))
        return out[: n.value]


_default_ctx = {}


def default_context(device: int = 0) -> Context:
    ctx = _default_ctx.get(device)
    if ctx is None:
        ctx = Context(device)
        _default_ctx[device] = ctx
    return ctx


def launch_count() -> int:
    return int(load_library().qtt_launch_count())


def dptr(a: np.ndarray):
    """ctypes double* of a C-contiguous float64 array."""
    return a.ctypes.data_as(_P)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)
