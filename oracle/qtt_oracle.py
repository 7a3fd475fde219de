"""numpy restatement of the reference QTT AMEn solve path -- TEST INFRASTRUCTURE.

Header (required by the build rules):
  * This module is the CPU *oracle* for parity tests and the CPU baseline leg of
    ``bench.py --impl reference``.  The product package never imports it.
  * It restates, in numpy + LAPACK (numpy.linalg / scipy.linalg), the algorithm
    of the reference package ``ttfem`` (pure Python, numpy/scipy):
      - ``/root/reference/pkg/src/ttfem/tt.py``   (containers, rounding, apply, norms)
      - ``/root/reference/pkg/src/ttfem/amen.py`` (the alternating sweep solver)
    Each function cites the reference ``file:line`` it follows.
  * Parity pin: ``tests/golden/make_golden.py`` imports the real reference in the
    build container and stores its outputs as ``tests/golden/*.npz``; the CPU test
    ``tests/test_oracle_golden.py`` checks this module against those fixtures.
  * Third-party algorithms the reference delegates to: LAPACK ``dgesdd``/``dgeqrf``/
    ``dpotrf`` via numpy 2.3 / scipy 1.18 (same calls are made here), and SciPy
    1.18 ``scipy.sparse.linalg.cg`` (restated below as :func:`pcg` from its
    published algorithm, so the GPU kernel mirrors an explicit recurrence).

Trains are plain Python lists of C-contiguous float64 arrays: vector cores
``(r_{k-1}, n_k, r_k)``, operator cores ``(R_{k-1}, m_k, n_k, R_k)``.
"""

from __future__ import annotations

import math
import time

import numpy as np
import scipy.linalg

__all__ = [
    "rank_for_tolerance", "orthogonalize_rl", "tt_round", "tt_apply", "tt_add",
    "tt_scale", "tt_sub", "tt_dot", "tt_norm", "tt_ones", "tt_zero", "tt_full",
    "op_full", "env_left", "env_right", "rhs_env_left", "rhs_env_right",
    "local_rhs", "local_matvec", "local_dense", "local_diag", "mixed_residual",
    "pcg", "solve_local", "truncated_factor", "default_x0", "probe_symmetry",
    "init_z", "residual_norm", "residual_norm_streaming", "amen_solve", "OracleSolverError",
]


class OracleSolverError(RuntimeError):
    """Mirror of ttfem.errors.SolverError (errors.py:29) for the oracle."""


# --------------------------------------------------------------------------
# tensor-train algebra   (reference: tt.py)
# --------------------------------------------------------------------------

def _ranks(cores):
    return [1] + [c.shape[-1] for c in cores]


def tt_ones(dims):
    """tt.py:221-222."""
    return [np.ones((1, n, 1)) for n in dims]


def tt_zero(dims):
    """tt.py:216-218 (canonical rank-1 zero)."""
    return [np.zeros((1, n, 1)) for n in dims]


def tt_full(cores):
    """Dense vector in big-endian C order (tt.py:276-283)."""
    acc = cores[0].reshape(cores[0].shape[1], cores[0].shape[2])
    for g in cores[1:]:
        acc = (acc @ g.reshape(g.shape[0], -1)).reshape(-1, g.shape[2])
    return acc.reshape(-1)


def op_full(cores):
    """Dense matrix of an operator train (tt.py:566-577)."""
    rows = int(np.prod([c.shape[1] for c in cores]))
    cols = int(np.prod([c.shape[2] for c in cores]))
    acc = np.ones((1, 1, 1))  # (rowsofar, colsofar, rank)
    for g in cores:
        r0, m, n, r1 = g.shape
        t = np.tensordot(acc, g, axes=(2, 0))  # (R, C, m, n, r1)
        t = t.transpose(0, 2, 1, 3, 4)
        acc = t.reshape(t.shape[0] * m, t.shape[2] * n, r1)
    return acc.reshape(rows, cols)


def tt_scale(cores, c):
    """tt.py:334-336: the scalar multiplies the first core only."""
    out = [np.array(g, dtype=np.float64, copy=True) for g in cores]
    out[0] = out[0] * float(c)
    return out


def tt_add(a, b):
    """Block concatenation, ranks add (tt.py:308-327)."""
    if len(a) == 1:
        return [a[0] + b[0]]
    out = []
    last = len(a) - 1
    for k, (ga, gb) in enumerate(zip(a, b)):
        if k == 0:
            out.append(np.concatenate([ga, gb], axis=2))
        elif k == last:
            out.append(np.concatenate([ga, gb], axis=0))
        else:
            blk = np.zeros((ga.shape[0] + gb.shape[0], ga.shape[1], ga.shape[2] + gb.shape[2]))
            blk[: ga.shape[0], :, : ga.shape[2]] = ga
            blk[ga.shape[0]:, :, ga.shape[2]:] = gb
            out.append(blk)
    return out


def tt_sub(a, b):
    """tt.py:330-331."""
    return tt_add(a, tt_scale(b, -1.0))


def tt_dot(a, b):
    """Gram contraction left to right (tt.py:351-359)."""
    w = np.ones((1, 1))
    for ga, gb in zip(a, b):
        t = np.tensordot(w, ga, axes=(0, 0))          # (rb, n, ra')
        w = np.tensordot(t, gb, axes=((0, 1), (0, 1)))  # (ra', rb')
    return float(w[0, 0])


def orthogonalize_rl(cores):
    """Right-to-left thin-QR sweep (tt.py:396-406).

    Core k is unfolded as (r_{k-1}, n r_k), transposed and QR-factored; Q^T
    becomes the new core, R^T is absorbed into core k-1.
    """
    g = [np.asarray(c, dtype=np.float64) for c in cores]
    for k in range(len(g) - 1, 0, -1):
        r0, n, r1 = g[k].shape
        q, rr = np.linalg.qr(g[k].reshape(r0, n * r1).T)
        g[k] = np.ascontiguousarray(q.T).reshape(q.shape[1], n, r1)
        g[k - 1] = np.tensordot(g[k - 1], rr.T, axes=(2, 0))
    return g


def tt_norm(cores):
    """Norm via orthogonalization (tt.py:362-371)."""
    if len(cores) == 1:
        return float(np.linalg.norm(cores[0]))
    return float(np.linalg.norm(orthogonalize_rl(cores)[0]))


def svd_thin(mat):
    """gesdd with gesvd fallback (tt.py:376-383)."""
    try:
        return np.linalg.svd(mat, full_matrices=False)
    except np.linalg.LinAlgError:
        return scipy.linalg.svd(mat, full_matrices=False, lapack_driver="gesvd")


def rank_for_tolerance(s, delta):
    """Smallest r >= 1 with ||s[r:]||_2 <= delta (tt.py:386-393).

    The tail norms are accumulated from the smallest singular value upwards
    with a sequential cumulative sum, exactly as the reference does, so the
    rank decision reproduces bit-for-bit given the same singular values.
    """
    s = np.asarray(s, dtype=np.float64)
    n = s.size
    if n == 0:
        return 1
    tails = np.sqrt(np.cumsum(s[::-1] ** 2))[::-1]  # tails[j] = ||s[j:]||
    r = n
    for j in range(n - 1, 0, -1):
        if tails[j] <= delta:
            r = j
        else:
            break
    return max(r, 1)


def tt_round(cores, rel_tolerance=1e-12, max_rank=None):
    """R->L orthogonalization then L->R truncated SVD (tt.py:409-429)."""
    K = len(cores)
    old = _ranks(cores)
    if K == 1 or all(r == 1 for r in old):
        return [np.array(c, copy=True) for c in cores]
    g = orthogonalize_rl(cores)
    nrm = float(np.linalg.norm(g[0]))
    if nrm == 0.0:
        return tt_zero([c.shape[1] for c in cores])
    delta = rel_tolerance * nrm / math.sqrt(K - 1)
    for k in range(K - 1):
        r0, n, r1 = g[k].shape
        u, s, vt = svd_thin(g[k].reshape(r0 * n, r1))
        keep = min(rank_for_tolerance(s, delta), old[k + 1])
        if max_rank is not None:
            keep = min(keep, max_rank)
        g[k] = u[:, :keep].reshape(r0, n, keep)
        g[k + 1] = np.tensordot(s[:keep, None] * vt[:keep], g[k + 1], axes=(1, 0))
    return g


def tt_apply(op, x):
    """Kronecker core products, no rounding (tt.py:434-449, policy=None)."""
    out = []
    for a, g in zip(op, x):
        ra0, m, n, ra1 = a.shape
        rx0, _, rx1 = g.shape
        # y[(a,x), m, (b,y)] = sum_n A[a,m,n,b] x[x,n,y]
        t = np.tensordot(a, g, axes=(2, 1))          # (ra0, m, ra1, rx0, rx1)
        t = t.transpose(0, 3, 1, 2, 4)                # (ra0, rx0, m, ra1, rx1)
        out.append(np.ascontiguousarray(t).reshape(ra0 * rx0, m, ra1 * rx1))
    return out


# --------------------------------------------------------------------------
# interface (environment) contractions   (reference: amen.py:102-160)
# --------------------------------------------------------------------------
# phi at a bond: (bra rank, operator rank, ket rank);  psi: (bra rank, rhs rank)

def env_left(phi, bra, a, ket):
    """phi'[U,B,Z] = sum phi[X,A,Y] ket[Y,n,Z] a[A,m,n,B] bra[X,m,U] (amen.py:108-111)."""
    t = np.tensordot(phi, ket, axes=(2, 0))               # X A n Z
    t = np.tensordot(t, a, axes=((1, 2), (0, 2)))         # X Z m B
    out = np.tensordot(bra, t, axes=((0, 1), (0, 2)))     # U Z B
    return np.ascontiguousarray(out.transpose(0, 2, 1))


def env_right(phi, bra, a, ket):
    """phi'[B,a,Y] = sum phi[X,A,Z] ket[Y,n,Z] a[a,m,n,A] bra[B,m,X] (amen.py:114-117)."""
    t = np.tensordot(ket, phi, axes=(2, 2))               # Y n X A
    t = np.tensordot(t, a, axes=((1, 3), (2, 3)))         # Y X a m
    out = np.tensordot(bra, t, axes=((1, 2), (3, 1)))     # B Y a
    return np.ascontiguousarray(out.transpose(0, 2, 1))


def rhs_env_left(psi, bra, f):
    """psi'[U,G] = sum psi[X,F] f[F,m,G] bra[X,m,U] (amen.py:120-122)."""
    t = np.tensordot(psi, f, axes=(1, 0))                 # X m G
    return np.tensordot(bra, t, axes=((0, 1), (0, 1)))    # U G


def rhs_env_right(psi, bra, f):
    """psi'[U,F] = sum psi[X,G] f[F,m,G] bra[U,m,X] (amen.py:125-127)."""
    t = np.tensordot(f, psi, axes=(2, 1))                 # F m X
    return np.tensordot(bra, t, axes=((1, 2), (1, 2)))    # U F


def local_rhs(psil, f, psir):
    """b[X,m,Y] = psil[X,F] f[F,m,G] psir[Y,G] (amen.py:130-131)."""
    t = np.tensordot(psil, f, axes=(1, 0))                # X m G
    return np.tensordot(t, psir, axes=(2, 1))             # X m Y


def local_matvec(phil, a, phir, v):
    """y[X,m,Y] = phil[X,a,U] v[U,n,V] A[a,m,n,b] phir[Y,b,V] (amen.py:134-137)."""
    t = np.tensordot(phil, v, axes=(2, 0))                # X a n V
    t = np.tensordot(t, a, axes=((1, 2), (0, 2)))         # X V m b
    return np.tensordot(t, phir, axes=((3, 1), (1, 2)))   # X m Y


def matvec_sweep(op, x):
    """Config-4 microbench from the reference's own primitives: right
    environments of x|A|x built right to left (amen.py:300-321 with _phi_right_step,
    amen.py:114), then for k = 0..K-1 y_k = _local_matvec(phi_L[k], A_k, phi_R[k+1], x_k)
    (amen.py:134) and phi_L[k+1] = _phi_left_step(phi_L[k], x_k, A_k, x_k) (amen.py:108)."""
    K = len(op)
    right = [None] * (K + 1)
    right[K] = np.ones((1, 1, 1))
    for k in range(K - 1, 0, -1):
        right[k] = env_right(right[k + 1], x[k], op[k], x[k])
    left = np.ones((1, 1, 1))
    ys = []
    for k in range(K):
        ys.append(local_matvec(left, op[k], right[k + 1], x[k]))
        if k + 1 < K:
            left = env_left(left, x[k], op[k], x[k])
    return ys


def local_dense(phil, a, phir):
    """Dense local matrix, rows (X,m,Y), cols (U,n,V) (amen.py:140-144)."""
    t = np.tensordot(phil, a, axes=(1, 0))                # X U m n b
    t = np.tensordot(t, phir, axes=(4, 1))                # X U m n Y V
    t = t.transpose(0, 2, 4, 1, 3, 5)                     # X m Y U n V
    dim = phil.shape[0] * a.shape[1] * phir.shape[0]
    return np.ascontiguousarray(t).reshape(dim, dim)


def local_diag(phil, a, phir):
    """Diagonal of the local matrix (amen.py:147-151)."""
    dp = np.diagonal(phil, axis1=0, axis2=2).T            # X a
    da = np.diagonal(a, axis1=1, axis2=2).transpose(0, 2, 1)  # a m b
    dq = np.diagonal(phir, axis1=0, axis2=2).T            # Y b
    t = np.tensordot(dp, da, axes=(1, 0))                 # X m b
    return np.tensordot(t, dq, axes=(2, 1))               # X m Y


def mixed_residual(psil, f, psir, phil, a, u, phir):
    """Projected f - A u (amen.py:154-160)."""
    return local_rhs(psil, f, psir) - local_matvec(phil, a, phir, u)


# --------------------------------------------------------------------------
# local solvers   (reference: amen.py:163-234)
# --------------------------------------------------------------------------

def pcg(matvec, b, x0, rtol, maxiter, inv_diag):
    """Jacobi-preconditioned CG, the recurrence of SciPy 1.18 ``cg``
    (scipy/sparse/linalg/_isolve/iterative.py) as called at amen.py:163-167
    with atol=0: stop when ||r|| < rtol*||b|| (checked before each step)."""
    b = np.asarray(b, dtype=np.float64).ravel()
    bnorm = float(np.linalg.norm(b))
    stop = max(0.0, rtol * bnorm)
    if bnorm == 0.0:
        return b.copy(), 0, 0
    x = np.array(x0, dtype=np.float64).ravel()
    r = b - matvec(x) if x.any() else b.copy()
    rho_old = None
    p = None
    for it in range(maxiter):
        if float(np.linalg.norm(r)) < stop:
            return x, 0, it
        z = r * inv_diag
        rho = float(np.dot(r, z))
        if it == 0:
            p = z.copy()
        else:
            p *= rho / rho_old
            p += z
        q = matvec(p)
        alpha = rho / float(np.dot(p, q))
        x += alpha * p
        r -= alpha * q
        rho_old = rho
    return x, maxiter, maxiter


def solve_local(phil, a, phir, rhs, prev, *, direct, direct_cap, tol, iter_cap, sweep, k):
    """amen.py:170-214.  Returns (u, lam, info) with info = dict(path, iters)."""
    dim = rhs.size
    if direct and dim <= direct_cap:
        mat = local_dense(phil, a, phir)
        try:
            fac = scipy.linalg.cho_factor(mat, lower=True)
        except np.linalg.LinAlgError as exc:
            raise OracleSolverError(
                f"local system not positive definite at sweep {sweep}, core {k} (dim {dim}): {exc}"
            ) from exc
        lam = float(np.abs(mat).sum(axis=1).max())
        u = scipy.linalg.cho_solve(fac, rhs.ravel()).reshape(rhs.shape)
        return u, lam, {"path": "direct", "iters": 0}
    dg = local_diag(phil, a, phir).ravel()
    lam = float(dg.sum())
    inv = 1.0 / np.where(dg > 0, dg, 1.0)
    shape = rhs.shape

    def mv(v):
        return local_matvec(phil, a, phir, v.reshape(shape)).ravel()

    u, info, its = pcg(mv, rhs.ravel(), prev.ravel(), max(0.05 * tol, 1e-13), iter_cap, inv)
    return u.reshape(shape), lam, {"path": "iterative", "iters": its}


def truncated_factor(mat, rel_tolerance, max_rank, delta_abs=None):
    """SVD split mat ~= Q W (amen.py:217-234)."""
    u, s, vt = np.linalg.svd(mat, full_matrices=False)
    total = float(np.linalg.norm(s))
    if total == 0.0:
        return u[:, :1], np.zeros((1, mat.shape[1]))
    delta = rel_tolerance * total
    if delta_abs is not None:
        delta = min(delta, delta_abs)
    r = rank_for_tolerance(s, delta)
    if max_rank is not None:
        r = min(r, max_rank)
    r = max(r, 1)
    return u[:, :r], s[:r, None] * vt[:r]


# --------------------------------------------------------------------------
# solver driver   (reference: amen.py:87-99, 237-510)
# --------------------------------------------------------------------------

def default_x0(op, f):
    """amen.py:237-246."""
    dims = [g.shape[1] for g in f]
    diag = [np.ascontiguousarray(np.diagonal(a, axis1=1, axis2=2).transpose(0, 2, 1)) for a in op]
    ones = tt_ones(dims)
    n = float(np.prod(dims))
    md = tt_dot(diag, ones) / n
    if abs(md) < 1e-300:
        return tt_round(f, 1e-12, 8)
    mf = tt_dot(f, ones) / n
    return tt_scale(ones, mf / md)


def probe_symmetry(op, rng):
    """Two random rank-2 probe pairs (amen.py:249-272); consumes rng draws."""
    dims = [a.shape[2] for a in op]
    K = len(dims)

    def draw():
        v = [rng.standard_normal((1 if k == 0 else 2, dims[k], 1 if k == K - 1 else 2))
             for k in range(K)]
        nv = tt_norm(v)
        return tt_scale(v, 1.0 / nv) if nv > 0 else v

    for _ in range(2):
        u, v = draw(), draw()
        au, av = tt_apply(op, u), tt_apply(op, v)
        s1, s2 = tt_dot(v, au), tt_dot(u, av)
        if abs(s1 - s2) > 1e-6 * (tt_norm(au) + tt_norm(av) + 1e-300):
            raise OracleSolverError("operator is not symmetric (<v,Au> != <u,Av> on random probes)")


def init_z(dims, rank, rng):
    """Random residual basis, right-orthogonalized (amen.py:275-284)."""
    K = len(dims)
    rk = [1] + [rank] * (K - 1) + [1]
    for k in range(1, K):
        rk[k] = min(rk[k], int(np.prod(dims[:k])), int(np.prod(dims[k:])))
    return orthogonalize_rl([rng.standard_normal((rk[k], dims[k], rk[k + 1])) for k in range(K)])


def residual_norm(op, x, f, rounding=None):
    """||A x - f|| / ||f|| (amen.py:87-99); rounding = (rel_tol, max_rank) or None."""
    r = tt_sub(tt_apply(op, x), f)
    if rounding is not None:
        r = tt_round(r, *rounding)
    nf, nr = tt_norm(f), tt_norm(r)
    return nr / nf if nf > 0 else nr


def residual_norm_streaming(op, x, f):
    """||A x - f|| / ||f|| exactly as residual_norm(op, x, f) with rounding=None (amen.py:87-99:
    tt_norm(tt_sub(tt_apply(A, x, None), f)), tt.py:330-336, 362-371, 396-406, 434-449), but
    with each difference core formed on the fly inside the right-to-left QR sweep, so the
    rank R*r + r_f train is never held whole (C5: ~45 GB if materialised).  Same cores, same
    LAPACK QR (dgeqrf; only R is used, so mode="r"), same absorption order."""
    K = len(op)

    def diff_core(k):
        y = tt_apply([op[k]], [x[k]])[0]
        g = f[k] * (-1.0 if k == 0 else 1.0)  # tt_scale(f, -1) scales the first core
        if K == 1:
            return y + g
        if k == 0:
            return np.concatenate([y, g], axis=2)
        if k == K - 1:
            return np.concatenate([y, g], axis=0)
        blk = np.zeros((y.shape[0] + g.shape[0], y.shape[1], y.shape[2] + g.shape[2]))
        blk[: y.shape[0], :, : y.shape[2]] = y
        blk[y.shape[0]:, :, y.shape[2]:] = g
        return blk

    carry = None
    for k in range(K - 1, 0, -1):
        core = diff_core(k)
        if carry is not None:
            core = np.tensordot(core, carry, axes=(2, 0))
        r0, n, r1 = core.shape
        rr = np.linalg.qr(core.reshape(r0, n * r1).T, mode="r")
        carry = rr.T
        del core
    core0 = diff_core(0)
    if carry is not None:
        core0 = np.tensordot(core0, carry, axes=(2, 0))
    nr = float(np.linalg.norm(core0))
    nf = tt_norm(f)
    return nr / nf if nf > 0 else nr


def _sweep(x, z, op, f, cfg, sweep, forward, state, stats):
    """One directional pass of amen.py:287-391; mutates x and z in place."""
    K = len(x)
    one3, one2 = np.ones((1, 1, 1)), np.ones((1, 1))
    Px = [None] * (K + 1)   # phi  (x|A|x)
    Pz = [None] * (K + 1)   # phiz (z|A|x)
    Qx = [None] * (K + 1)   # psi  (x|f)
    Qz = [None] * (K + 1)   # psiz (z|f)
    for env in (Px, Pz):
        env[0], env[K] = one3, one3
    for env in (Qx, Qz):
        env[0], env[K] = one2, one2
    if forward:
        for k in range(K - 1, 0, -1):
            Px[k] = env_right(Px[k + 1], x[k], op[k], x[k])
            Qx[k] = rhs_env_right(Qx[k + 1], x[k], f[k])
            Pz[k] = env_right(Pz[k + 1], z[k], op[k], x[k])
            Qz[k] = rhs_env_right(Qz[k + 1], z[k], f[k])
        order = range(K)
    else:
        for k in range(K - 1):
            Px[k + 1] = env_left(Px[k], x[k], op[k], x[k])
            Qx[k + 1] = rhs_env_left(Qx[k], x[k], f[k])
            Pz[k + 1] = env_left(Pz[k], z[k], op[k], x[k])
            Qz[k + 1] = rhs_env_left(Qz[k], z[k], f[k])
        order = range(K - 1, -1, -1)

    est = 0.0
    for k in order:
        rl, m, rr = x[k].shape
        b = local_rhs(Qx[k], f[k], Qx[k + 1])
        u, lam, info = solve_local(
            Px[k], op[k], Px[k + 1], b, x[k], direct=cfg["local_solver"] == "direct",
            direct_cap=cfg["direct_dim_cap"], tol=cfg["residual_tol"],
            iter_cap=cfg["local_iter_cap"], sweep=sweep, k=k)
        if stats is not None:
            stats.append((sweep, k, rl, m, rr, info["path"], info["iters"]))
        state["lam_max"] = max(state["lam_max"], lam)
        dabs = None
        if K > 1 and state["lam_max"] > 0:
            dabs = cfg["residual_tol"] * state["f_norm"] / (state["lam_max"] * math.sqrt(K - 1))
        zeta = mixed_residual(Qz[k], f[k], Qz[k + 1], Pz[k], op[k], u, Pz[k + 1])
        if (forward and k == K - 1) or (not forward and k == 0):
            x[k] = u
            z[k] = zeta
            est = float(np.linalg.norm(zeta))
            break
        rel, cap = cfg["rounding"]
        if forward:
            enr = mixed_residual(Qx[k], f[k], Qz[k + 1], Px[k], op[k], u, Pz[k + 1])
            qf, w = truncated_factor(u.reshape(rl * m, rr), rel, cap, dabs)
            q, rmat = np.linalg.qr(np.hstack([qf, enr.reshape(rl * m, -1)]))
            x[k] = q.reshape(rl, m, q.shape[1])
            x[k + 1] = np.tensordot(rmat[:, : qf.shape[1]] @ w, x[k + 1], axes=(1, 0))
            zq, _ = np.linalg.qr(zeta.reshape(zeta.shape[0] * m, -1))
            z[k] = zq.reshape(zeta.shape[0], m, zq.shape[1])
            Px[k + 1] = env_left(Px[k], x[k], op[k], x[k])
            Qx[k + 1] = rhs_env_left(Qx[k], x[k], f[k])
            Pz[k + 1] = env_left(Pz[k], z[k], op[k], x[k])
            Qz[k + 1] = rhs_env_left(Qz[k], z[k], f[k])
        else:
            enr = mixed_residual(Qz[k], f[k], Qx[k + 1], Pz[k], op[k], u, Px[k + 1])
            qf, w = truncated_factor(u.reshape(rl, m * rr).T, rel, cap, dabs)
            q, rmat = np.linalg.qr(np.hstack([qf, enr.reshape(-1, m * rr).T]))
            x[k] = np.ascontiguousarray(q.T).reshape(q.shape[1], m, rr)
            x[k - 1] = np.tensordot(x[k - 1], (rmat[:, : qf.shape[1]] @ w).T, axes=(2, 0))
            zq, _ = np.linalg.qr(zeta.reshape(-1, m * zeta.shape[2]).T)
            z[k] = np.ascontiguousarray(zq.T).reshape(zq.shape[1], m, zeta.shape[2])
            Px[k] = env_right(Px[k + 1], x[k], op[k], x[k])
            Qx[k] = rhs_env_right(Qx[k + 1], x[k], f[k])
            Pz[k] = env_right(Pz[k + 1], z[k], op[k], x[k])
            Qz[k] = rhs_env_right(Qz[k + 1], z[k], f[k])
    return est


DEFAULT_CONFIG = {
    # amen.py:48-64 defaults
    "residual_tol": 1e-8,
    "max_sweeps": 50,
    "enrichment_rank": 4,
    "local_solver": "direct",
    "direct_dim_cap": 4096,
    "local_iter_cap": 400,
    "rounding": (1e-10, 80),
    "seed": 2024,
    "stagnation_strikes": 3,
}


def amen_solve(op, f, x0=None, config=None, stats=None, sweep_hook=None):
    """amen.py:394-510.  Returns (x cores, report dict).

    ``stats`` (optional list) collects one tuple per local solve;
    ``sweep_hook(sweep, x)`` (optional) may return True to stop early -- used
    only by the bounded CPU-baseline sample in bench.py.
    """
    cfg = dict(DEFAULT_CONFIG)
    cfg.update(config or {})
    dims = [g.shape[1] for g in f]
    t0 = time.perf_counter()
    nf = tt_norm(f)
    if nf == 0.0:
        return tt_zero(dims), {"converged": True, "sweeps_used": 0,
                               "final_relative_residual": 0.0, "rank_profile_history": (),
                               "wall_time": time.perf_counter() - t0, "residual_history": ()}
    rng = np.random.default_rng(cfg["seed"])
    probe_symmetry(op, rng)
    start = x0 if x0 is not None else default_x0(op, f)
    x = orthogonalize_rl(start)
    if tt_norm(x) == 0.0:
        x = orthogonalize_rl(tt_scale(tt_ones(dims), nf))
    z = init_z(dims, cfg["enrichment_rank"], rng)
    check = (0.1 * cfg["residual_tol"], None)
    state = {"lam_max": 0.0, "f_norm": nf}
    ranks_hist, res_hist = [], []
    converged, final = False, None
    best, strikes, last_check = math.inf, 0, -10
    tol = cfg["residual_tol"]
    for sweep in range(1, cfg["max_sweeps"] + 1):
        est = _sweep(x, z, op, f, cfg, sweep, sweep % 2 == 1, state, stats)
        ranks_hist.append(tuple(_ranks(x)))
        res_hist.append(est / nf)
        if sweep_hook is not None and sweep_hook(sweep, x):
            break
        cert = est / nf <= tol
        plateau = (cfg["stagnation_strikes"] > 0 and len(res_hist) >= 8
                   and min(res_hist[-4:]) > 0.97 * min(res_hist[-8:-4]))
        spaced = sweep - last_check >= 5
        if not cert and not (plateau and spaced):
            continue
        final = residual_norm(op, x, f, check)
        if final <= tol:
            converged = True
            break
        if not cert and spaced:
            if final > 0.97 * best:
                strikes += 1
                if strikes >= cfg["stagnation_strikes"]:
                    break
                z[:] = init_z(dims, cfg["enrichment_rank"], rng)
            else:
                strikes = 0
            last_check = sweep
        best = min(best, final)
    if final is None or not converged:
        final = residual_norm(op, x, f, check)
        converged = final <= tol
    return x, {"converged": bool(converged), "sweeps_used": len(ranks_hist),
               "final_relative_residual": float(final),
               "rank_profile_history": tuple(ranks_hist),
               "wall_time": time.perf_counter() - t0, "residual_history": tuple(res_hist)}
