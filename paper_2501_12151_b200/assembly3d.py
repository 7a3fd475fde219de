"""3D Q1 linear-elasticity assembly in serial-binary QTT layout (host side).

This is the *caller* that feeds the hot path, not
the hot path itself.  The reference only assembles 2D plane stress
(``/root/reference/pkg/src/ttfem/elasticity.py:522-667``); BASELINE.json's
configs are 3D, so this module supplies the equivalent 3D operator with the same
conventions:

* 2^L nodes per axis (2^L - 1 trilinear cells), grid.py:63-77;
* dof ordering (component, x, y, z) with the component core first
  (grid.py:318-323) and *serial* binary digits per axis, most significant first
  (tt.py:194-200): cores = [component (mode 3)] + L x-digits + L y-digits + L z-digits;
* symmetric clamp  A = P A_raw P + (I - P),  f = P (M f0)   (elasticity.py:559-565, 612-620);
* solver scaling by the mean diagonal of P A_raw P (elasticity.py:629-667).

The stiffness is an exact sum of Kronecker products of 1D Q1 matrices
(stiffness K1, mass M1, first-derivative coupling C1), one (1,3,3,1) component
core in front.  Material E may vary per z-element layer (config C5); the
z-factor of every term is then assembled with the layer's E (exact piecewise
integration, the layer interface may cut an element).  Everything is host
numpy: assembly runs once per problem, outside the timed solve.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["ElasticityProblem", "assemble_cube", "lame_3d", "stiffness_qtt"]


def lame_3d(E, nu):
    """3D Lame constants (lambda, mu)."""
    return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


# ---------------------------------------------------------------- 1D element integrals

_G2 = (np.array([-1.0, 1.0]) / math.sqrt(3.0) + 1.0) / 2.0  # Gauss 2-pt on [0,1]


def _element_matrices_1d(N, weight_fn, lo=0.0, hi=1.0):
    """Exact 1D Q1 matrices on N uniform nodes of [lo, hi] with a piecewise
    constant weight w(t) (called at the midpoint of each sub-interval).

    Returns (K, M, C) with K = int w phi_i' phi_j', M = int w phi_i phi_j,
    C = int w phi_i' phi_j.  Elements cut by a weight discontinuity are
    split at the breakpoints the weight function reports.
    """
    h = (hi - lo) / (N - 1)
    K = np.zeros((N, N))
    M = np.zeros((N, N))
    C = np.zeros((N, N))
    for e in range(N - 1):
        a, b = lo + e * h, lo + (e + 1) * h
        cuts = [a] + [c for c in weight_fn.breaks if a < c < b] + [b]
        for s0, s1 in zip(cuts[:-1], cuts[1:]):
            w = weight_fn((s0 + s1) / 2.0)
            for g in _G2:
                t = s0 + g * (s1 - s0)
                wq = (s1 - s0) / 2.0 * w
                phi = np.array([(b - t) / h, (t - a) / h])
                dphi = np.array([-1.0 / h, 1.0 / h])
                idx = [e, e + 1]
                for i in range(2):
                    for j in range(2):
                        K[idx[i], idx[j]] += wq * dphi[i] * dphi[j]
                        M[idx[i], idx[j]] += wq * phi[i] * phi[j]
                        C[idx[i], idx[j]] += wq * dphi[i] * phi[j]
    return K, M, C


class _Const:
    breaks: tuple = ()

    def __init__(self, v=1.0):
        self.v = v

    def __call__(self, t):
        return self.v


class _Layers:
    """E = e_lo for t < cut, e_hi for t >= cut."""

    def __init__(self, cut, e_lo, e_hi):
        self.breaks = (cut,)
        self.cut, self.e_lo, self.e_hi = cut, e_lo, e_hi

    def __call__(self, t):
        return self.e_lo if t < self.cut else self.e_hi


def _patch_load_1d(N, lo, hi):
    """g[i] = int_{lo}^{hi} phi_i(t) dt on N uniform nodes of [0,1] (exact)."""
    h = 1.0 / (N - 1)
    g = np.zeros(N)
    for e in range(N - 1):
        a, b = e * h, (e + 1) * h
        s0, s1 = max(a, lo), min(b, hi)
        if s1 <= s0:
            continue
        for q in _G2:
            t = s0 + q * (s1 - s0)
            wq = (s1 - s0) / 2.0
            g[e] += wq * (b - t) / h
            g[e + 1] += wq * (t - a) / h
    return g


# ---------------------------------------------------------------- tiny host TT toolbox
# (assembly-time only; the solve path's TT algebra lives on the device)

def _svd_compress(tensor, dims, tol):
    """TT-SVD of a dense tensor with modes ``dims``; relative Frobenius tol."""
    K = len(dims)
    nrm = float(np.linalg.norm(tensor))
    delta = tol * nrm / math.sqrt(max(K - 1, 1))
    cores, rest, rp = [], tensor.reshape(1, -1), 1
    for k in range(K - 1):
        mat = rest.reshape(rp * dims[k], -1)
        u, s, vt = np.linalg.svd(mat, full_matrices=False)
        tail = np.sqrt(np.cumsum(s[::-1] ** 2))[::-1]
        r = len(s)
        while r > 1 and tail[r - 1] <= delta:
            r -= 1
        cores.append(u[:, :r].reshape(rp, dims[k], r))
        rest = s[:r, None] * vt[:r]
        rp = r
    cores.append(rest.reshape(rp, dims[-1], 1))
    return cores


def _matrix_qtt(mat, L, tol=1e-15):
    """QTT operator cores (r,2,2,r) of an 2^L x 2^L matrix, big-endian digits."""
    t = mat.reshape([2] * (2 * L))
    perm = [ax for k in range(L) for ax in (k, L + k)]
    fused = t.transpose(perm).reshape([4] * L)
    cores = _svd_compress(fused, [4] * L, tol)
    return [c.reshape(c.shape[0], 2, 2, c.shape[2]) for c in cores]


def _vector_qtt(vec, L, tol=1e-15):
    return _svd_compress(vec.reshape([2] * L), [2] * L, tol)


def _op_add(A, B):
    if len(A) == 1:
        return [A[0] + B[0]]
    out = []
    for k, (a, b) in enumerate(zip(A, B)):
        if k == 0:
            out.append(np.concatenate([a, b], axis=3))
        elif k == len(A) - 1:
            out.append(np.concatenate([a, b], axis=0))
        else:
            c = np.zeros((a.shape[0] + b.shape[0], a.shape[1], a.shape[2], a.shape[3] + b.shape[3]))
            c[: a.shape[0], :, :, : a.shape[3]] = a
            c[a.shape[0]:, :, :, a.shape[3]:] = b
            out.append(c)
    return out


def _op_sum(trains):
    """Sum of operator trains: the block-diagonal cores that folding `_op_add` over the list
    builds, allocated once (the fold re-copies the growing sum per term: 2.4 of the 4.4 s of the
    C3 assembly)."""
    if len(trains) == 1:
        return list(trains[0])
    K = len(trains[0])
    if K == 1:
        acc = trains[0][0]
        for t in trains[1:]:
            acc = acc + t[0]
        return [acc]
    # all cores live back to back in ONE buffer: DeviceTrain.upload then sends it as it is
    # (the 21-term C3 sum is 1.45 GB; gathering its cores into an upload buffer cost 0.3 s)
    shapes = []
    for k in range(K):
        cs = [t[k] for t in trains]
        if k == 0:
            shapes.append((1, cs[0].shape[1], cs[0].shape[2], sum(c.shape[3] for c in cs)))
        elif k == K - 1:
            shapes.append((sum(c.shape[0] for c in cs), cs[0].shape[1], cs[0].shape[2], 1))
        else:
            shapes.append((sum(c.shape[0] for c in cs), cs[0].shape[1], cs[0].shape[2],
                           sum(c.shape[3] for c in cs)))
    flat = np.zeros(sum(int(np.prod(sh)) for sh in shapes))
    out, off = [], 0
    for k, sh in enumerate(shapes):
        n = int(np.prod(sh))
        c = flat[off:off + n].reshape(sh)
        off += n
        i = j = 0
        for t in trains:
            b = t[k]
            if k == 0:
                c[:, :, :, j:j + b.shape[3]] = b
            elif k == K - 1:
                c[i:i + b.shape[0]] = b
            else:
                c[i:i + b.shape[0], :, :, j:j + b.shape[3]] = b
            i += b.shape[0]
            j += b.shape[3]
        out.append(c)
    return out


def _op_compose(A, B):
    """(A @ B) cores: apply B first."""
    out = []
    for a, b in zip(A, B):
        t = np.tensordot(a, b, axes=(2, 1))  # ra0 m ra1 rb0 n rb1
        t = t.transpose(0, 3, 1, 4, 2, 5)
        s = t.shape
        out.append(np.ascontiguousarray(t).reshape(s[0] * s[1], s[2], s[3], s[4] * s[5]))
    return out


def _orth_rl(cores):
    g = list(cores)
    for k in range(len(g) - 1, 0, -1):
        r0 = g[k].shape[0]
        rest = g[k].shape[1:]
        q, r = np.linalg.qr(g[k].reshape(r0, -1).T)
        g[k] = np.ascontiguousarray(q.T).reshape((q.shape[1],) + rest)
        g[k - 1] = np.tensordot(g[k - 1], r.T, axes=(g[k - 1].ndim - 1, 0))
    return g


def _op_round(A, tol):
    """Round an operator train as a fused-mode vector (like tt.py:506-531)."""
    if len(A) == 1:
        return A
    shapes = [(c.shape[1], c.shape[2]) for c in A]
    vec = [c.reshape(c.shape[0], -1, c.shape[3]) for c in A]
    g = _orth_rl(vec)
    nrm = float(np.linalg.norm(g[0]))
    delta = tol * nrm / math.sqrt(len(g) - 1)
    for k in range(len(g) - 1):
        r0, n, r1 = g[k].shape
        u, s, vt = np.linalg.svd(g[k].reshape(r0 * n, r1), full_matrices=False)
        tail = np.sqrt(np.cumsum(s[::-1] ** 2))[::-1]
        r = len(s)
        while r > 1 and tail[r - 1] <= delta:
            r -= 1
        g[k] = u[:, :r].reshape(r0, n, r)
        g[k + 1] = np.tensordot(s[:r, None] * vt[:r], g[k + 1], axes=(1, 0))
    return [c.reshape(c.shape[0], m, n, c.shape[2]) for c, (m, n) in zip(g, shapes)]


def _op_scale(A, c):
    out = [x.copy() for x in A]
    out[0] = out[0] * c
    return out


def _op_diag_mean(A):
    """mean of the diagonal of an operator train."""
    w = np.ones((1,))
    total = 1
    for c in A:
        d = np.einsum("ammb->ab", c)
        w = w @ d
        total *= c.shape[1]
    return float(w[0]) / total


def _apply(A, x):
    out = []
    for a, g in zip(A, x):
        t = np.tensordot(a, g, axes=(2, 1))  # ra0 m ra1 rx0 rx1
        t = t.transpose(0, 3, 1, 2, 4)
        s = t.shape
        out.append(np.ascontiguousarray(t).reshape(s[0] * s[1], s[2], s[3] * s[4]))
    return out


def _vec_round(x, tol):
    g = _orth_rl(x)
    nrm = float(np.linalg.norm(g[0]))
    if nrm == 0.0 or len(g) == 1:
        return g
    delta = tol * nrm / math.sqrt(len(g) - 1)
    for k in range(len(g) - 1):
        r0, n, r1 = g[k].shape
        u, s, vt = np.linalg.svd(g[k].reshape(r0 * n, r1), full_matrices=False)
        tail = np.sqrt(np.cumsum(s[::-1] ** 2))[::-1]
        r = len(s)
        while r > 1 and tail[r - 1] <= delta:
            r -= 1
        g[k] = u[:, :r].reshape(r0, n, r)
        g[k + 1] = np.tensordot(s[:r, None] * vt[:r], g[k + 1], axes=(1, 0))
    return g


def _scale_vec(x, c):
    out = [g.copy() for g in x]
    out[0] = out[0] * c
    return out


# ---------------------------------------------------------------- assembly

@dataclass
class ElasticityProblem:
    """Solver-ready system: ``op`` and ``rhs`` are lists of numpy cores.

    op cores are (R, m, n, R); rhs cores are (r, n, r).  ``scale`` is the mean
    diagonal the elastic block and load were divided by (elasticity.py:654-667).
    """

    L: int
    op: list
    rhs: list
    scale: float
    dims: tuple
    description: dict

    @property
    def op_ranks(self):
        return (1,) + tuple(c.shape[3] for c in self.op)

    @property
    def dof(self):
        return 3 * 8 ** self.L


def _comp_core(a, b, coef):
    c = np.zeros((1, 3, 3, 1))
    c[0, a, b, 0] = coef
    return c


def _factors(L, E=1.0, layers=None):
    """1D factor QTTs (K, M, C, C^T): x/y axes with unit weight, the z axis carries E(z)."""
    N = 2 ** L
    wz = _Layers(*layers) if layers is not None else _Const(E)
    K1, M1, C1 = _element_matrices_1d(N, _Const(1.0))
    Kz, Mz, Cz = _element_matrices_1d(N, wz)
    q = {
        ("K", 0): _matrix_qtt(K1, L), ("M", 0): _matrix_qtt(M1, L),
        ("C", 0): _matrix_qtt(C1, L), ("Ct", 0): _matrix_qtt(C1.T.copy(), L),
        ("K", 2): _matrix_qtt(Kz, L), ("M", 2): _matrix_qtt(Mz, L),
        ("C", 2): _matrix_qtt(Cz, L), ("Ct", 2): _matrix_qtt(Cz.T.copy(), L),
    }
    return lambda kind, axis: q[(kind, 2 if axis == 2 else 0)]


def _rounders(rounding):
    """(operator rounding, vector rounding) at a relative tolerance: "device" runs the
    engine's tt_round (tt.py:409-429 semantics; R->L Householder QR, L->R one-sided Jacobi SVD
    on the B200 -- deterministic on every B200), "host" the numpy restatement above (its
    noise-level cuts at 1e-14 depend on the host's BLAS threading)."""
    if rounding == "host":
        return _op_round, _vec_round
    if rounding != "device":
        raise ValueError(f"rounding must be 'device' or 'host', got {rounding!r}")
    from . import tt as T

    def op(A, tol):
        if len(A) == 1:
            return A
        return [np.ascontiguousarray(c) for c in T.tt_op_round(T.TTLinearOperator(A), T.TruncationPolicy(tol)).cores]

    def vec(x, tol):
        return [np.ascontiguousarray(c) for c in T.tt_round(T.TensorTrain(x), T.TruncationPolicy(tol)).cores]

    return op, vec


def stiffness_qtt(L, nu=0.3, E=1.0, layers=None, round_tol=1e-14, factor=None, rounding="host"):
    """Unclamped Q1 stiffness of the unit cube as a QTT operator (component core first,
    serial binary digits): the exact sum of 21 Kronecker terms, rounded at round_tol."""
    lam1, mu1 = lame_3d(1.0, nu)  # per unit E; E enters through the weights
    factor = factor or _factors(L, E, layers)
    op_round, _ = _rounders(rounding)

    def D(p, r):
        """int d_p phi_i d_r phi_j as per-axis factors."""
        kinds = []
        for ax in range(3):
            if ax == p and ax == r:
                kinds.append("K")
            elif ax == p:
                kinds.append("C")
            elif ax == r:
                kinds.append("Ct")
            else:
                kinds.append("M")
        return kinds

    terms = []  # (a, b, coef, kinds)
    for a in range(3):
        for b in range(3):
            if a != b:
                terms.append((a, b, lam1, D(a, b)))
                terms.append((a, b, mu1, D(b, a)))
            else:
                terms.append((a, a, lam1 + 2.0 * mu1, D(a, a)))
                for c in range(3):
                    if c != a:
                        terms.append((a, a, mu1, D(c, c)))
    trains = []
    for a, b, coef, kinds in terms:
        cores = [_comp_core(a, b, coef)]
        for ax in range(3):
            cores += list(factor(kinds[ax], ax))
        trains.append(cores)
    return op_round(_op_sum(trains), round_tol)


def assemble_cube(L, nu=0.3, E=1.0, layers=None, load="body", body=(0.0, 0.0, -1.0),
                  traction=(0.0, 0.0, -1.0), patch=(0.25, 0.75), round_tol=1e-14, rounding="device"):
    """Clamped unit cube (x = 0 face fixed), E, nu, serial binary QTT.

    layers:   None (uniform E) or (cut_z, E_lo, E_hi) -- E depends on z only.
    load:     "body"  -> constant body force ``body`` through the consistent mass;
              "patch" -> traction ``traction`` on the x = 1 face patch y,z in ``patch``.
    rounding: where the round_tol roundings of the operator and load trains run (the
              reference rounds its assembled operator with tt_op_round, elasticity.py:557-565):
              "device" (the engine's tt_round; needs the B200) or "host" (numpy, for CPU-only
              tooling such as the reference-ensemble scripts).
    """
    if L < 1:
        raise ValueError("L must be >= 1")
    N = 2 ** L
    factor = _factors(L, E, layers)
    _op_round, _vec_round = _rounders(rounding)
    A_raw = stiffness_qtt(L, nu, E, layers, round_tol, factor, rounding)

    # clamp projector P = I3 (x) diag(1 - e0) (x) I (x) I     (x = 0 face)
    eye2 = np.eye(2).reshape(1, 2, 2, 1)
    e00 = np.zeros((1, 2, 2, 1))
    e00[0, 0, 0, 0] = 1.0
    px = _op_add([eye2.copy() for _ in range(L)], _op_scale([e00.copy() for _ in range(L)], -1.0))
    P = [np.eye(3).reshape(1, 3, 3, 1)] + px + [eye2.copy() for _ in range(2 * L)]
    I_full = [np.eye(3).reshape(1, 3, 3, 1)] + [eye2.copy() for _ in range(3 * L)]
    PAP = _op_round(_op_compose(_op_compose(P, A_raw), P), round_tol)
    scale = _op_diag_mean(PAP)
    if not scale > 0:
        raise ValueError("non-positive mean diagonal")
    A = _op_round(_op_add(_op_scale(PAP, 1.0 / scale), _op_add(I_full, _op_scale(P, -1.0))), round_tol)

    # load vector
    if load == "body":
        f0 = [np.asarray(body, dtype=np.float64).reshape(1, 3, 1)] + [np.ones((1, 2, 1)) for _ in range(3 * L)]
        M3 = [np.eye(3).reshape(1, 3, 3, 1)]
        for ax in range(3):
            M3 += [c.copy() for c in factor("M", ax)]
        f = _apply(M3, f0)
    elif load == "patch":
        g = _patch_load_1d(N, *patch)
        ex = np.zeros(N)
        ex[N - 1] = 1.0
        f = ([np.asarray(traction, dtype=np.float64).reshape(1, 3, 1)]
             + _vector_qtt(ex, L) + _vector_qtt(g, L) + _vector_qtt(g, L))
    else:
        raise ValueError(f"unknown load {load!r}")
    f = _vec_round(_apply(P, f), round_tol)
    f = _scale_vec(f, 1.0 / scale)
    desc = {"L": L, "nu": nu, "E": E, "layers": layers, "load": load, "layout": "serial-binary",
            "dof": 3 * N ** 3, "cells_per_axis": N - 1, "round_tol": round_tol, "rounding": rounding}
    return ElasticityProblem(L=L, op=A, rhs=f, scale=scale, dims=(3,) + (2,) * (3 * L),
                             description=desc)
