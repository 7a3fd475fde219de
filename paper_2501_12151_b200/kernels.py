"""Host wrappers of the device interface contractions (K1-K4 of SURVEY.md 2.3).

Same names, argument order and layouts as the reference's private helpers in
``ttfem/amen.py:108-160`` (which ``ttfem.amen`` re-exports under underscore names):
    _phi_left_step(phi, xb, ac, xk)      amen.py:108
    _phi_right_step(phi, xb, ac, xk)     amen.py:114
    _psi_left_step(psi, xb, fc)          amen.py:120
    _psi_right_step(psi, xb, fc)         amen.py:125
    _local_rhs(psil, fc, psir)           amen.py:130
    _local_matvec(phil, ac, phir, v)     amen.py:134
    _local_dense(phil, ac, phir)         amen.py:140
    _local_diag(phil, ac, phir)          amen.py:147
    _mixed_residual(...)                 amen.py:154
Each call copies its numpy inputs to the device, runs the sm_100a kernels and
returns a fresh numpy array (inputs are never mutated).
"""
from __future__ import annotations

import numpy as np

from . import _native as nat
from .errors import ShapeMismatchError


def _ctx(ctx):
    return ctx if ctx is not None else nat.default_context()


def _need(cond, msg):
    if not cond:
        raise ShapeMismatchError(msg)


def local_matvec(phil, ac, phir, v, ctx=None):
    phil, ac, phir, v = (nat.f64(a) for a in (phil, ac, phir, v))
    rX, Ra, rU = phil.shape
    _need(ac.ndim == 4 and ac.shape[0] == Ra, f"operator core {ac.shape} vs phil {phil.shape}")
    _, m, n, Rb = ac.shape
    rY, Rb2, rV = phir.shape
    _need(Rb2 == Rb and v.shape == (rU, n, rV), f"local matvec shapes {phil.shape} {ac.shape} {phir.shape} {v.shape}")
    y = np.empty((rX, m, rY))
    nat.call("qtt_local_matvec", _ctx(ctx).handle, nat.dptr(phil), nat.dptr(ac), nat.dptr(phir),
             nat.dptr(v), rX, Ra, rU, m, n, Rb, rY, rV, nat.dptr(y))
    return y


def phi_left_step(phi, xb, ac, xk, ctx=None):
    phi, xb, ac, xk = (nat.f64(a) for a in (phi, xb, ac, xk))
    rX, RA, rY = phi.shape
    _, m, n, RB = ac.shape
    rU = xb.shape[2]
    rZ = xk.shape[2]
    _need(xb.shape[:2] == (rX, m) and xk.shape[:2] == (rY, n) and ac.shape[0] == RA,
          f"env left shapes {phi.shape} {xb.shape} {ac.shape} {xk.shape}")
    out = np.empty((rU, RB, rZ))
    nat.call("qtt_env_left", _ctx(ctx).handle, nat.dptr(phi), nat.dptr(xb), nat.dptr(ac), nat.dptr(xk),
             rX, RA, rY, m, n, RB, rU, rZ, nat.dptr(out))
    return out


def phi_right_step(phi, xb, ac, xk, ctx=None):
    phi, xb, ac, xk = (nat.f64(a) for a in (phi, xb, ac, xk))
    rX, RA, rZ = phi.shape
    Ra, m, n, RA2 = ac.shape
    rB = xb.shape[0]
    rY = xk.shape[0]
    _need(RA2 == RA and xb.shape[1:] == (m, rX) and xk.shape[1:] == (n, rZ),
          f"env right shapes {phi.shape} {xb.shape} {ac.shape} {xk.shape}")
    out = np.empty((rB, Ra, rY))
    nat.call("qtt_env_right", _ctx(ctx).handle, nat.dptr(phi), nat.dptr(xb), nat.dptr(ac), nat.dptr(xk),
             rX, RA, rZ, m, n, Ra, rB, rY, nat.dptr(out))
    return out


def psi_left_step(psi, xb, fc, ctx=None):
    psi, xb, fc = (nat.f64(a) for a in (psi, xb, fc))
    rX, rF = psi.shape
    _, m, rG = fc.shape
    rU = xb.shape[2]
    _need(fc.shape[0] == rF and xb.shape[:2] == (rX, m), f"psi left shapes {psi.shape} {xb.shape} {fc.shape}")
    out = np.empty((rU, rG))
    nat.call("qtt_psi_left", _ctx(ctx).handle, nat.dptr(psi), nat.dptr(xb), nat.dptr(fc),
             rX, rF, m, rU, rG, nat.dptr(out))
    return out


def psi_right_step(psi, xb, fc, ctx=None):
    psi, xb, fc = (nat.f64(a) for a in (psi, xb, fc))
    rX, rG = psi.shape
    rF, m, _ = fc.shape
    rU = xb.shape[0]
    _need(fc.shape[2] == rG and xb.shape[1:] == (m, rX), f"psi right shapes {psi.shape} {xb.shape} {fc.shape}")
    out = np.empty((rU, rF))
    nat.call("qtt_psi_right", _ctx(ctx).handle, nat.dptr(psi), nat.dptr(xb), nat.dptr(fc),
             rX, rG, rU, m, rF, nat.dptr(out))
    return out


def local_rhs(psil, fc, psir, ctx=None):
    psil, fc, psir = (nat.f64(a) for a in (psil, fc, psir))
    rX, rF = psil.shape
    _, m, rG = fc.shape
    rY = psir.shape[0]
    _need(fc.shape[0] == rF and psir.shape[1] == rG, f"local rhs shapes {psil.shape} {fc.shape} {psir.shape}")
    out = np.empty((rX, m, rY))
    nat.call("qtt_local_rhs", _ctx(ctx).handle, nat.dptr(psil), nat.dptr(fc), nat.dptr(psir),
             rX, rF, m, rG, rY, nat.dptr(out))
    return out


def local_dense(phil, ac, phir, ctx=None):
    phil, ac, phir = (nat.f64(a) for a in (phil, ac, phir))
    rX, Ra, rU = phil.shape
    _, m, n, Rb = ac.shape
    rY, _, rV = phir.shape
    out = np.empty((rX * m * rY, rU * n * rV))
    nat.call("qtt_local_dense", _ctx(ctx).handle, nat.dptr(phil), nat.dptr(ac), nat.dptr(phir),
             rX, Ra, rU, m, n, Rb, rY, rV, nat.dptr(out))
    return out


def local_diag(phil, ac, phir, ctx=None):
    phil, ac, phir = (nat.f64(a) for a in (phil, ac, phir))
    rX, Ra, _ = phil.shape
    _, m, _, Rb = ac.shape
    rY = phir.shape[0]
    out = np.empty((rX, m, rY))
    nat.call("qtt_local_diag", _ctx(ctx).handle, nat.dptr(phil), nat.dptr(ac), nat.dptr(phir),
             rX, Ra, m, Rb, rY, nat.dptr(out))
    return out


def mixed_residual(psil, fc, psir, phil, ac, u, phir, ctx=None):
    psil, fc, psir, phil, ac, u, phir = (nat.f64(a) for a in (psil, fc, psir, phil, ac, u, phir))
    rX, rF = psil.shape
    _, m, rG = fc.shape
    rY = psir.shape[0]
    _, Ra, rU = phil.shape
    _, _, n, Rb = ac.shape
    rV = phir.shape[2]
    out = np.empty((rX, m, rY))
    nat.call("qtt_mixed_residual", _ctx(ctx).handle, nat.dptr(psil), nat.dptr(fc), nat.dptr(psir),
             nat.dptr(phil), nat.dptr(ac), nat.dptr(u), nat.dptr(phir),
             rX, rF, rG, rY, Ra, rU, m, n, Rb, rV, nat.dptr(out))
    return out


SWEEP_TIME_FIELDS = ("prepass_ms", "sweep_ms", "k1_ms", "k2_ms", "k1_flops", "k2_flops", "prepass_flops")


def matvec_sweep(A, x, ctx=None, timing=False, split_timing=False, return_y=True):
    """Config-4 microbench operation: right-environment pre-pass, then one
    left-to-right sweep of ``_local_matvec(phi_L[k], A_k, phi_R[k+1], x_k)`` (amen.py:134)
    followed by ``_phi_left_step(phi_L[k], x_k, A_k, x_k)`` (amen.py:108), all on the device.

    A / x: TTLinearOperator / TensorTrain (uploaded) or DeviceTrain handles (resident).
    Returns (list of y_k cores or None, dict of CUDA-event times/flops or None)."""
    import ctypes

    from .tt import DeviceTrain
    ctx = _ctx(ctx)
    dA = A if isinstance(A, DeviceTrain) else DeviceTrain.upload(A.cores, ctx)
    dx = x if isinstance(x, DeviceTrain) else DeviceTrain.upload(x.cores, ctx)
    h = ctypes.c_void_p()
    times = np.zeros(len(SWEEP_TIME_FIELDS))
    nat.call("qtt_matvec_sweep", ctx.handle, dA.handle, dx.handle, 1 if split_timing else 0,
             ctypes.byref(h) if return_y else None, nat.dptr(times) if timing else None)
    ys = DeviceTrain(h, ctx).cores() if return_y else None
    return ys, (dict(zip(SWEEP_TIME_FIELDS, times.tolist())) if timing else None)
