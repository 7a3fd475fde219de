"""Alternating-sweep (AMEn) TT solver -- drop-in for ``ttfem.amen`` (amen.py).

``amen_solve`` keeps the reference signature (amen.py:394) and returns the same
``(TensorTrain, SolveReport)``; the whole sweep loop runs on the B200 inside
libqtt.so (csrc/amen.cu): environments stay resident in HBM across sweeps, local
systems are solved by a device Cholesky (dim <= direct_dim_cap) or a device
Jacobi-PCG with SciPy's stopping rule, truncations use a device Jacobi SVD with
the reference rank rule.  The random streams of ``np.random.default_rng(seed)``
(symmetry probes, residual bases, re-draws on stagnation strikes) are generated
here, in the reference's order, and consumed by the device solver, so both sides
see identical random numbers.

The private kernels of the reference module are re-exported with the same names
and argument order for the parity harness (``_local_matvec``, ``_phi_left_step``...).
"""
from __future__ import annotations

import ctypes
import logging
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from . import kernels as _k
from .errors import ShapeMismatchError
from .tt import (
    DeviceTrain,
    TensorTrain,
    TTLinearOperator,
    TruncationPolicy,
    _orthogonalize_rl,
    _rank_for_tolerance,
    tt_zero,
)

log = logging.getLogger(__name__)

__all__ = ["AmenConfig", "SolveReport", "amen_solve", "residual_norm"]

DIRECT = "direct"
ITERATIVE = "iterative"

# Local CG engine: 1 = one persistent cooperative kernel per local solve (default),
# 0 = per-step kernel launches (kept for A/B measurements).
FUSED_CG = int(os.environ.get("QTT_FUSED_CG", "1"))

# reference private helpers, same names (amen.py:108-160)
_phi_left_step = _k.phi_left_step
_phi_right_step = _k.phi_right_step
_psi_left_step = _k.psi_left_step
_psi_right_step = _k.psi_right_step
_local_rhs = _k.local_rhs
_local_matvec = _k.local_matvec
_local_dense = _k.local_dense
_local_diag = _k.local_diag
_mixed_residual = _k.mixed_residual
__all_private__ = (_orthogonalize_rl, _rank_for_tolerance)


@dataclass(frozen=True)
class AmenConfig:
    """Solver knobs, same fields and defaults as amen.py:48-74."""

    residual_tol: float = 1e-8
    max_sweeps: int = 50
    enrichment_rank: int = 4
    local_solver: str = DIRECT
    direct_dim_cap: int = 4096
    local_iter_cap: int = 400
    rounding: TruncationPolicy = TruncationPolicy(rel_tolerance=1e-10, max_rank=80)
    seed: int = 2024
    stagnation_strikes: int = 3

    def __post_init__(self):
        if self.residual_tol <= 0:
            raise ValueError("residual_tol must be > 0")
        if self.enrichment_rank < 1 or self.max_sweeps < 1:
            raise ValueError("enrichment_rank and max_sweeps must be >= 1")
        if self.local_solver not in (DIRECT, ITERATIVE):
            raise ValueError(f"unknown local_solver {self.local_solver!r}")
        if self.stagnation_strikes < 0:
            raise ValueError("stagnation_strikes must be >= 0")


@dataclass(frozen=True)
class SolveReport:
    """amen.py:77-84."""

    converged: bool
    sweeps_used: int
    final_relative_residual: float
    rank_profile_history: tuple
    wall_time: float
    residual_history: tuple


def residual_norm(A, x, f, rounding=None, ctx=None):
    """Relative residual ||A x - f|| / ||f|| (absolute when ||f|| = 0), amen.py:87-99.

    Same semantics as the reference: with ``rounding=None`` the norm of the unrounded
    difference train A x - f, taken on the device by the exact QR sweep over its
    Kronecker-structured cores (no rank R*r + r_f train is materialised); with a
    ``rounding`` policy, A x - f is formed (device tt_apply), rounded with that policy
    (device tt_round) and its norm taken, as amen.py:95-98 does.

    (amen_solve's own certifications use the unrounded exact norm: rounding at
    0.1*tol is a sequence of orthogonal projections, so it moves the norm by at most
    0.1*tol relative -- DESIGN.md section 4.)
    """
    if A.col_dims != x.dims or A.row_dims != f.dims:
        raise ShapeMismatchError(
            f"operator {A.row_dims}x{A.col_dims} does not fit x dims {x.dims}, f dims {f.dims}")
    ctx = ctx or nat.default_context()
    if rounding is not None:
        from .tt import tt_apply, tt_norm, tt_round, tt_sub
        r = tt_round(tt_sub(tt_apply(A, x, None, ctx=ctx), f), rounding, ctx=ctx)
        nf = tt_norm(f, ctx=ctx)
        nr = tt_norm(r, ctx=ctx)
        return nr / nf if nf > 0 else nr
    dA, dx, df = DeviceTrain.upload(A.cores, ctx), DeviceTrain.upload(x.cores, ctx), DeviceTrain.upload(f.cores, ctx)
    out, used = ctypes.c_double(), ctypes.c_int()
    nat.call("qtt_residual_norm", ctx.handle, dA.handle, dx.handle, df.handle, 0, ctypes.byref(out),
             ctypes.byref(used))
    return float(out.value)


def random_draws(A: TTLinearOperator, dims, config: AmenConfig) -> np.ndarray:
    """The standard-normal stream ``amen_solve`` consumes, in the reference's order:
    two probe pairs (amen.py:249-272), the first z basis (amen.py:275-284, 429) and
    the re-draws after stagnation strikes (amen.py:485)."""
    rng = np.random.default_rng(config.seed)
    K = len(dims)
    parts = []
    for _ in range(2):
        for _vec in range(2):
            for k, n in enumerate(A.col_dims):
                r0 = 1 if k == 0 else 2
                r1 = 1 if k == K - 1 else 2
                parts.append(rng.standard_normal((r0, n, r1)).ravel())
    ranks = [1] + [config.enrichment_rank] * (K - 1) + [1]
    for k in range(1, K):
        ranks[k] = min(ranks[k], int(np.prod(dims[:k])), int(np.prod(dims[k:])))
    # a strike can happen at most once per sweep (strikes reset on progress), so
    # 1 + max_sweeps basis draws always cover the solve; unused draws are ignored
    n_sets = 1 + (config.max_sweeps if config.stagnation_strikes > 0 else 0)
    for _ in range(n_sets):
        for k in range(K):
            parts.append(rng.standard_normal((ranks[k], dims[k], ranks[k + 1])).ravel())
    return np.ascontiguousarray(np.concatenate(parts), dtype=np.float64)


def _params(config: AmenConfig) -> nat.AmenParams:
    p = nat.AmenParams()
    p.residual_tol = config.residual_tol
    p.max_sweeps = config.max_sweeps
    p.enrichment_rank = config.enrichment_rank
    p.local_iterative = 1 if config.local_solver == ITERATIVE else 0
    p.direct_dim_cap = config.direct_dim_cap
    p.local_iter_cap = config.local_iter_cap
    p.round_tol = config.rounding.rel_tolerance
    p.round_max_rank = 0 if config.rounding.max_rank is None else config.rounding.max_rank
    p.stagnation_strikes = config.stagnation_strikes
    p.fused_cg = FUSED_CG
    return p


def amen_solve_device(dA: DeviceTrain, df: DeviceTrain, dx0, config: AmenConfig, draws: np.ndarray,
                      K: int, ctx):
    """Solve with device-resident inputs; returns (DeviceTrain x, report fields)."""
    rep = nat.AmenReport()
    rank_hist = np.zeros((config.max_sweeps, K + 1), dtype=np.int32)
    res_hist = np.zeros(config.max_sweeps)
    h = ctypes.c_void_p()
    prm = _params(config)
    nat.call("qtt_amen_solve", ctx.handle, dA.handle, df.handle, dx0.handle if dx0 is not None else None,
             ctypes.byref(prm), nat.dptr(draws), int(draws.size), ctypes.byref(h), ctypes.byref(rep),
             rank_hist.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), nat.dptr(res_hist))
    n = rep.sweeps_used
    info = {
        "converged": bool(rep.converged),
        "sweeps_used": n,
        "final_relative_residual": float(rep.final_relative_residual),
        "rank_profile_history": tuple(tuple(int(v) for v in row) for row in rank_hist[:n]),
        "residual_history": tuple(float(v) for v in res_hist[:n]),
        "certifications_gram": rep.certifications_gram,
        "certifications_exact": rep.certifications_exact,
    }
    return DeviceTrain(h, ctx), info


def amen_solve(A, f, x0=None, config=None, ctx=None):
    """Solve A x = f in TT form on the device; returns (x, SolveReport) (amen.py:394)."""
    config = config or AmenConfig()
    if not isinstance(A, TTLinearOperator):
        raise ShapeMismatchError("A must be a TT linear operator")
    if A.row_dims != A.col_dims:
        raise ShapeMismatchError(f"A is not square: {A.row_dims} x {A.col_dims}")
    if A.col_dims != f.dims:
        raise ShapeMismatchError(f"operator columns {A.col_dims} do not match f dims {f.dims}")
    if x0 is not None and x0.dims != f.dims:
        raise ShapeMismatchError(f"x0 dims {x0.dims} do not match f {f.dims}")
    ctx = ctx or nat.default_context()
    t0 = time.perf_counter()
    draws = random_draws(A, f.dims, config)
    dA = DeviceTrain.upload(A.cores, ctx)
    df = DeviceTrain.upload(f.cores, ctx)
    dx0 = DeviceTrain.upload(x0.cores, ctx) if x0 is not None else None
    dx, info = amen_solve_device(dA, df, dx0, config, draws, A.order, ctx)
    x = TensorTrain(dx.cores())
    if info["sweeps_used"] == 0 and info["converged"]:
        x = tt_zero(f.dims)
    wall = time.perf_counter() - t0
    if not info["converged"] and info["sweeps_used"] < config.max_sweeps:
        log.warning("residual stagnated at %.3e (tolerance %.1e); stopping",
                    info["final_relative_residual"], config.residual_tol)
    tail = info["residual_history"][-3:]
    if info["converged"] and len(tail) == 3 and not (tail[0] >= tail[1] >= tail[2]):
        log.warning("residual estimates not monotone over the final sweeps: %s", list(tail))
    report = SolveReport(
        converged=info["converged"],
        sweeps_used=info["sweeps_used"],
        final_relative_residual=info["final_relative_residual"],
        rank_profile_history=info["rank_profile_history"],
        wall_time=wall,
        residual_history=info["residual_history"],
    )
    return x, report


def _core_step(A: TTLinearOperator, f: TensorTrain, config: AmenConfig, sweep: int, k: int, forward: bool,
               lam_max: float, f_norm: float, state, ctx=None):
    """One core step of ``_sweep`` (amen.py:324-390) run by the engine's own per-core code on
    injected state (qtt_amen_step) -- the state-injected parity check.  ``state`` holds the
    11 arrays x_k, x_nb, z_k, phi_k, phi_k1, phiz_k, phiz_k1, psi_k, psi_k1, psiz_k, psiz_k1
    (psi as (bra, rhs) or (bra, rhs, 1)); returns (outputs, info): the new x_k, x_nb, z_k and
    phi/phiz/psi/psiz at the rebuilt bond, and {"lam", "rank", "iters"}."""
    ctx = ctx or nat.default_context()
    arrs = [nat.f64(a.reshape(a.shape + (1,) * (3 - a.ndim))) for a in state]
    if len(arrs) != 11:
        raise ValueError("the core step takes 11 state arrays")
    ptrs = (nat._P * 11)(*[nat.dptr(a) for a in arrs])
    dims = np.array([d for a in arrs for d in a.shape], dtype=np.int64)
    dA, df = DeviceTrain.upload(A.cores, ctx), DeviceTrain.upload(f.cores, ctx)
    h = ctypes.c_void_p()
    lam, rank, iters = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
    prm = _params(config)
    nat.call("qtt_amen_step", ctx.handle, dA.handle, df.handle, ctypes.byref(prm), int(sweep), int(k),
             1 if forward else 0, float(lam_max), float(f_norm), 11, ptrs,
             dims.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.byref(h), ctypes.byref(lam),
             ctypes.byref(rank), ctypes.byref(iters))
    outs = DeviceTrain(h, ctx).cores()
    return outs, {"lam": float(lam.value), "rank": int(rank.value), "iters": int(iters.value)}

