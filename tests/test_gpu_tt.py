"""GPU parity of the dense factorizations (K6/K7), TT algebra (K9/K10, rounding)
and the local solvers (K4/K5) against the reference fixtures and the oracle."""
import ctypes
import os

import numpy as np
import pytest

from oracle import qtt_oracle as O
from tests.golden_io import load, train

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def tt():
    from paper_2501_12151_b200 import tt as T
    return T


@pytest.mark.parametrize("shape", [(1, 1), (5, 3), (3, 5), (64, 32), (200, 104), (130, 130), (7, 300)])
def test_qr_matches_numpy(tt, shape):
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    a = rng.standard_normal(shape)
    q, r = tt._qr(a)
    qn, rn = np.linalg.qr(a)
    assert rel(q @ r, a) <= 1e-13
    # LAPACK dlarfg sign convention reproduced -> factors equal, not just up to signs
    assert rel(q, qn) <= 1e-12 and rel(r, rn) <= 1e-12
    k = min(shape)
    assert np.linalg.norm(q.T @ q - np.eye(k)) <= 1e-13 * k


@pytest.mark.parametrize("shape", [(600, 300), (2100, 1030), (300, 900)])
def test_qr_large_matches_numpy(tt, shape):
    """Past one CTA's shared memory: blocked multi-CTA QR (geqrf + dorgqr), LAPACK signs."""
    rng = np.random.default_rng(shape[0] + shape[1])
    a = rng.standard_normal(shape)
    q, r = tt._qr(a)
    qn, rn = np.linalg.qr(a)
    assert rel(q @ r, a) <= 1e-13
    assert rel(q, qn) <= 1e-11 and rel(r, rn) <= 1e-12
    k = min(shape)
    assert np.linalg.norm(q.T @ q - np.eye(k)) <= 1e-13 * k


@pytest.mark.parametrize("shape,grade", [((700, 300), 10), ((1300, 1100), 12), ((520, 520), 0), ((300, 800), 6)])
def test_svd_large_matches_numpy(tt, shape, grade):
    """Block one-sided Jacobi (multi-CTA) on graded and flat spectra.  Like LAPACK gesdd
    (tt.py:376-383) the factorization is backward stable: singular values to eps * s_max,
    U s Vt to eps * ||a||, U orthonormal.  The rows of Vt come from normalized Jacobi columns,
    so rows of singular values s << s_max are orthonormal only to ~eps * s_max / s: checked
    on the rows with s >= 1e-3 s_max (the products S Vt used downstream are accurate)."""
    rng = np.random.default_rng(shape[0] * 3 + shape[1])
    a = rng.standard_normal(shape) * np.logspace(0, -grade, shape[1])[None, :]
    u, s, vt = tt._svd(a)
    sn = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(s - sn)) <= 1e-13 * sn[0]
    assert rel(u @ np.diag(s) @ vt, a) <= 5e-13  # backward error ~ eps sqrt(n) x sweeps
    k = min(shape)
    big = int(np.sum(s >= 1e-3 * s[0]))
    if shape[0] >= shape[1]:
        assert np.linalg.norm(u.T @ u - np.eye(k)) <= 1e-12 * k
        assert np.linalg.norm(vt[:big] @ vt[:big].T - np.eye(big)) <= 1e-12 * k
    else:  # wide: factored as the transpose, roles of U and Vt swap
        assert np.linalg.norm(vt @ vt.T - np.eye(k)) <= 1e-12 * k
        assert np.linalg.norm(u[:, :big].T @ u[:, :big] - np.eye(big)) <= 1e-12 * k


@pytest.mark.parametrize("shape", [(50, 20), (120, 100)])
def test_svd_rank_deficient(tt, shape):
    """Exactly rank-5 input: zero singular values come out as (near) zero, U still
    orthonormal (Jacobi columns of norm zero map to unit basis vectors)."""
    rng = np.random.default_rng(shape[1])
    a = rng.standard_normal((shape[0], 5)) @ rng.standard_normal((5, shape[1]))
    u, s, vt = tt._svd(a)
    sn = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(s - sn)) <= 1e-13 * sn[0]
    assert rel(u @ np.diag(s) @ vt, a) <= 1e-13
    k = min(shape)
    assert np.linalg.norm(u.T @ u - np.eye(k)) <= 1e-12 * k


def test_qr_rank_deficient(tt):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((40, 5)) @ rng.standard_normal((5, 12))
    q, r = tt._qr(a)
    assert rel(q @ r, a) <= 1e-13
    z = np.zeros((6, 4))
    q, r = tt._qr(z)
    qn, rn = np.linalg.qr(z)
    assert np.array_equal(r, rn) and rel(q, qn) == 0.0


@pytest.mark.parametrize("shape", [(1, 1), (8, 3), (3, 8), (72, 36), (200, 100), (150, 150), (30, 120),
                                   (16, 16), (40, 17), (100, 45), (64, 64), (180, 75), (96, 96), (224, 112),
                                   (300, 101), (113, 113)])
def test_svd_matches_numpy(tt, shape):
    """Covers every width bucket of the square-Jacobi kernel (n = 16 K, K = 1..7) and both
    neighbours of its range.  Widths whose one-CTA working set does not fit shared memory
    (here 150) take the block Jacobi, whose Vt rows for s << s_max are orthonormal only to
    ~eps * s_max / s (see test_svd_large_matches_numpy): checked on s >= 1e-3 s_max there."""
    rng = np.random.default_rng(shape[0] + 1000 * shape[1])
    a = rng.standard_normal(shape) * np.logspace(0, -10, shape[1])[None, :]
    u, s, vt = tt._svd(a)
    sn = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(s - sn)) <= 1e-13 * sn[0]
    assert rel(u @ np.diag(s) @ vt, a) <= 1e-13
    k = min(shape)
    one_cta = 2 * k * k + k <= 27 * 1024
    big = k if one_cta else int(np.sum(s >= 1e-3 * s[0]))
    if shape[0] >= shape[1]:
        assert np.linalg.norm(u.T @ u - np.eye(k)) <= 1e-12 * k
        assert np.linalg.norm(vt[:big] @ vt[:big].T - np.eye(big)) <= 1e-12 * k
    else:
        assert np.linalg.norm(vt @ vt.T - np.eye(k)) <= 1e-12 * k
        assert np.linalg.norm(u[:, :big].T @ u[:, :big] - np.eye(big)) <= 1e-12 * k


def test_svd_two_cta_jacobi_same_bits_as_one_cta():
    """The 2-CTA Jacobi (W and its angles in one CTA, V one DSMEM hop behind in the other,
    linalg.cu jacobi_sq2_kernel) performs the floating-point operations of the one-CTA kernel in
    the same order: U, s, Vt equal bit for bit.  (QTT_JAC_SQ2 is read once per process: one
    child process per setting; 3 = every width the cluster kernel supports, 0 = never.)"""
    import subprocess
    import sys
    code = (
        "import sys, hashlib, numpy as np\n"
        "sys.path.insert(0, %r)\n"
        "from paper_2501_12151_b200 import tt\n"
        "h = hashlib.sha256()\n"
        "for m, n in [(200, 100), (100, 100), (224, 112), (96, 81), (130, 65), (90, 40), (70, 33)]:\n"
        "    rng = np.random.default_rng(m * 7 + n)\n"
        "    a = rng.standard_normal((m, n)) * np.logspace(0, -8, n)[None, :]\n"
        "    for x in tt._svd(a):\n"
        "        h.update(np.ascontiguousarray(x).tobytes())\n"
        "print(h.hexdigest())\n"
    ) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for setting in ("0", "3"):
        env = dict(os.environ, QTT_JAC_SQ2=setting)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[setting] = r.stdout.strip().splitlines()[-1]
    assert out["0"] == out["3"], out


def test_truncated_factor_ranks_vs_reference(tt):
    """K6: the device SVD + rank rule reproduce the reference's rank decisions."""
    d = load("factor.npz")
    for i in range(int(d["tf_count"])):
        mat = d[f"tf{i}_mat"]
        rel_tol, cap, dabs = d[f"tf{i}_pol"]
        u, s, vt = tt._svd(mat)
        norm = float(np.linalg.norm(s))
        if norm == 0.0:
            r = 1
            qw = np.zeros_like(mat)
        else:
            delta = rel_tol * norm
            if dabs >= 0:
                delta = min(delta, dabs)
            r = tt._rank_for_tolerance(s, delta)
            if cap >= 0:
                r = min(r, int(cap))
            r = max(r, 1)
            qw = u[:, :r] @ (s[:r, None] * vt[:r])
        assert r == int(d[f"tf{i}_rank"]), i
        assert np.linalg.norm(qw - d[f"tf{i}_qw"]) <= 1e-12 * max(1.0, np.linalg.norm(d[f"tf{i}_qw"]))
    for j in range(int(d["rr_count"])):
        assert tt._rank_for_tolerance(d[f"rr{j}_s"], float(d[f"rr{j}_delta"])) == int(d[f"rr{j}_r"])


def test_tt_algebra_vs_reference(tt):
    d = load("tt_ops.npz")
    v, w, A = (train(d, n) for n in ("v", "w", "A"))
    orth = tt._orthogonalize_rl(v)
    ref = train(d, "v_orth")
    assert [c.shape for c in orth] == [c.shape for c in ref]
    for c, r in zip(orth, ref):  # same Householder signs -> same cores
        assert rel(c, r) <= 1e-12
    V, W = tt.TensorTrain(v), tt.TensorTrain(w)
    assert abs(tt.tt_norm(V) - float(d["v_norm"])) <= 1e-13 * float(d["v_norm"])
    assert abs(tt.tt_dot(V, W) - float(d["vw_dot"])) <= 1e-12 * abs(float(d["vw_dot"]))
    S = tt.tt_add(V, W)
    for j in range(4):
        tol, cap = d[f"round{j}_pol"]
        out = tt.tt_round(S, tt.TruncationPolicy(float(tol), None if cap < 0 else int(cap)))
        refj = train(d, f"round{j}")
        assert [c.shape for c in out.cores] == [c.shape for c in refj], j
        assert rel(O.tt_full(out.cores), O.tt_full(refj)) <= 1e-12
    dbl = tt.tt_round(tt.tt_add(V, V))
    assert [c.shape for c in dbl.cores] == [c.shape for c in train(d, "round_double")]
    Aop = tt.TTLinearOperator(A)
    av = tt.tt_apply(Aop, V, None)
    for c, r in zip(av.cores, train(d, "Av")):
        assert c.shape == r.shape and rel(c, r) <= 1e-15
    avr = tt.tt_apply(Aop, V, tt.TruncationPolicy(1e-8))
    assert [c.shape for c in avr.cores] == [c.shape for c in train(d, "Av_round")]
    assert rel(O.tt_full(avr.cores), O.tt_full(train(d, "Av_round"))) <= 1e-8


def test_residual_norm_vs_reference(tt):
    from paper_2501_12151_b200.amen import residual_norm
    d = load("tt_ops.npz")
    V, W = tt.TensorTrain(train(d, "v")), tt.TensorTrain(train(d, "w"))
    A = tt.TTLinearOperator(train(d, "A"))
    r = residual_norm(A, V, W)
    assert abs(r - float(d["resid_none"])) <= 1e-10 * float(d["resid_none"])
    r2 = residual_norm(A, V, W, tt.TruncationPolicy(1e-9))
    assert abs(r2 - float(d["resid_round"])) <= 1e-8 * float(d["resid_round"])


def test_local_solve_vs_reference():
    from paper_2501_12151_b200 import _native as nat
    d = load("solve_local.npz")
    phil, A, phir, rhs, prev = (nat.f64(d[k]) for k in ("phil", "Ak", "phir", "rhs", "prev"))
    rl, R0, _ = phil.shape
    _, m, _, R1 = A.shape
    rr = phir.shape[0]
    ctx = nat.default_context()
    cases = [(0, 1e-8, "direct", 1), (1, 1e-8, "iter_u_1e-08", 0), (1, 1e-4, "iter_u_0.0001", 0),
             (1, 1e-8, "iter_u_1e-08", 1), (1, 1e-4, "iter_u_0.0001", 1)]
    for iterative, tol, key, fused in cases:
        u = np.empty((rl, m, rr))
        lam, its = ctypes.c_double(), ctypes.c_int()
        nat.call("qtt_local_solve", ctx.handle, nat.dptr(phil), nat.dptr(A), nat.dptr(phir), nat.dptr(rhs),
                 nat.dptr(prev), rl, R0, m, R1, rr, iterative, 4096, tol, 400, fused, nat.dptr(u),
                 ctypes.byref(lam), ctypes.byref(its))
        if key == "direct":
            assert rel(u, d["direct_u"]) <= 1e-12
            assert abs(lam.value - float(d["direct_lam"])) <= 1e-12 * float(d["direct_lam"])
        else:
            # not bitwise (summation order): within the CG tolerance of the same recurrence
            assert rel(u, d[key]) <= max(10 * 0.05 * tol, 1e-11)
            lam_ref = float(d[key.replace("_u_", "_lam_")])
            assert abs(lam.value - lam_ref) <= 1e-12 * abs(lam_ref)


# shapes: small; C2 full rank; then the C3 x-rank 100 at operator ranks that take the fragment-run
# dealing of the CG kernel's first GEMM phase through 1, 2, 4, 6 and 10 fragments per warp; an
# unequal-rank system; and a C5-size system (rank 196, operator rank 52) whose per-CTA share
# exceeds one region, i.e. the row-block dealing with several regions per CTA (no oracle: 5 GFLOP
# per CPU matvec)
@pytest.mark.parametrize("rl,R,rr", [(12, 7, 9), (40, 20, 36), (68, 49, 68), (100, 5, 100), (100, 9, 100),
                                     (100, 17, 100), (100, 31, 100), (100, 52, 100), (96, 40, 100),
                                     (196, 52, 196)])
def test_fused_cg_matches_stepwise_cg(rl, R, rr):
    """The persistent cooperative CG kernel runs the same recurrence as the
    per-step path and the oracle's SciPy-cg restatement on an SPD local system."""
    from paper_2501_12151_b200 import _native as nat
    rng = np.random.default_rng(rl * 100 + rr)
    m = 2
    # SPD environments: Gram matrices per operator slice, SPD operator core
    gl = rng.standard_normal((R, rl, rl))
    phil = np.einsum("aij,akj->iak", gl, gl) / rl + np.eye(rl)[:, None, :]
    gr = rng.standard_normal((R, rr, rr))
    phir = np.einsum("aij,akj->iak", gr, gr) / rr + np.eye(rr)[:, None, :]
    G = rng.standard_normal((R, m, m, R)) / R
    A = np.einsum("amnb,apnb->ampb", G, G)  # symmetric PSD in (m, p) per (a, b)
    A = nat.f64(A + 0.5 * np.einsum("ab,mn->amnb", np.eye(R), np.eye(m)))
    phil, phir = nat.f64(phil), nat.f64(phir)
    rhs = nat.f64(rng.standard_normal((rl, m, rr)))
    prev = nat.f64(rng.standard_normal((rl, m, rr)) * 0.1)
    ctx = nat.default_context()
    outs = []
    for fused in (0, 1):
        u = np.empty((rl, m, rr))
        lam, its = ctypes.c_double(), ctypes.c_int()
        nat.call("qtt_local_solve", ctx.handle, nat.dptr(phil), nat.dptr(A), nat.dptr(phir), nat.dptr(rhs),
                 nat.dptr(prev), rl, R, m, R, rr, 1, 4096, 1e-6, 400, fused, nat.dptr(u),
                 ctypes.byref(lam), ctypes.byref(its))
        outs.append((u.copy(), its.value, lam.value))
    (u0, i0, l0), (u1, i1, l1) = outs
    assert abs(i0 - i1) <= 1
    assert rel(u1, u0) <= 1e-9
    assert abs(l0 - l1) <= 1e-12 * abs(l0)
    if rl > 100:
        return
    uo, lo, info = O.solve_local(phil, A, phir, rhs, prev, direct=False, direct_cap=4096, tol=1e-6,
                                 iter_cap=400, sweep=1, k=0)
    assert rel(u1, uo) <= 1e-8 and abs(info["iters"] - i1) <= 1


@pytest.mark.parametrize("L,r", [(2, 6), (3, 12), (5, 16)])
def test_residual_norm_structured_sweep_vs_oracle(L, r):
    """Certification norm (structured Kronecker cores + blocked Householder QR) vs the
    oracle's tt_norm(tt_sub(tt_apply(A, x), f)) on the 3D cube operator; multi-panel QRs
    at L=5 (unfoldings up to ~1500 x 750)."""
    from paper_2501_12151_b200.amen import residual_norm
    from paper_2501_12151_b200.assembly3d import assemble_cube
    from paper_2501_12151_b200.tt import TensorTrain, TTLinearOperator
    prob = assemble_cube(L)
    rng = np.random.default_rng(L * 10 + r)
    dims = prob.dims
    K = len(dims)
    ranks = [1] + [min(r, int(np.prod(dims[:k])), int(np.prod(dims[k:]))) for k in range(1, K)] + [1]
    x = [rng.standard_normal((ranks[k], dims[k], ranks[k + 1])) / np.sqrt(ranks[k]) for k in range(K)]
    ref = O.residual_norm(prob.op, x, prob.rhs)
    got = residual_norm(TTLinearOperator(prob.op), TensorTrain(x), TensorTrain(prob.rhs))
    assert abs(got - ref) <= 1e-11 * ref


def test_dense_bridges_vs_oracle(tt):
    """tt_to_dense (GEMM chain) and batched tt_entry on the device against the oracle's
    contraction (tt.py:276-298), including the leading 3-component mode."""
    rng = np.random.default_rng(11)
    dims = (3, 2, 2, 2, 2, 2, 2, 2)
    ranks = [1, 3, 5, 7, 6, 4, 5, 2, 1]
    cores = [rng.standard_normal((ranks[k], dims[k], ranks[k + 1])) for k in range(len(dims))]
    t = tt.TensorTrain(cores)
    full = tt.tt_to_dense(t)
    ref = O.tt_full(cores)
    assert rel(full, ref) <= 1e-14
    idx = np.stack([rng.integers(0, d, size=50) for d in dims], axis=1)
    got = tt.tt_entries(t, idx)
    flat = np.ravel_multi_index(tuple(idx.T), dims)
    assert np.max(np.abs(got - ref[flat])) <= 1e-13 * np.max(np.abs(ref))
    assert abs(tt.tt_entry(t, list(idx[0])) - ref[flat[0]]) <= 1e-13 * np.max(np.abs(ref))
    with pytest.raises(ValueError):
        tt.tt_entry(t, [3] + [0] * (len(dims) - 1))


def test_op_round_vs_reference(tt):
    """tt_op_round over fused (row, col) modes (tt.py:506-531): ranks and dense operator equal
    to the reference's, for a rank-doubled stiffness (A + A) and a capped random operator."""
    d = load("op_round.npz")
    for name, pol in (("AA", tt.TruncationPolicy(1e-10)), ("B", tt.TruncationPolicy(1e-2, 3))):
        out = tt.tt_op_round(tt.TTLinearOperator(train(d, name)), pol)
        ref = train(d, f"{name}_round")
        assert [c.shape for c in out.cores] == [c.shape for c in ref], name
        assert rel(O.op_full(list(out.cores)), O.op_full(ref)) <= 1e-12, name


def test_op_to_dense_vs_oracle(tt):
    """tt_op_to_dense via the device contraction of the fused-mode train (tt.py:566-577)."""
    d = load("op_round.npz")
    A = train(d, "AA_round")
    assert rel(tt.tt_op_to_dense(tt.TTLinearOperator(A)), O.op_full(A)) <= 1e-14


def test_round_edge_cases_vs_oracle(tt):
    """tt_round's special cases (tt.py:409-429): order 1 and all-ranks-1 trains return an
    unchanged copy, the zero train becomes the canonical rank-1 zero, max_rank caps after the
    tolerance, ranks never grow; tt_apply rejects mismatched modes."""
    from paper_2501_12151_b200.errors import ShapeMismatchError
    rng = np.random.default_rng(3)
    one = [rng.standard_normal((1, 4, 1))]
    out = tt.tt_round(tt.TensorTrain(one))
    assert len(out.cores) == 1 and np.array_equal(out.cores[0], one[0])
    r1 = [rng.standard_normal((1, 2, 1)) for _ in range(5)]
    out = tt.tt_round(tt.TensorTrain(r1))
    assert all(np.array_equal(a, b) for a, b in zip(out.cores, r1))
    z = [np.zeros((1, 2, 3)), np.zeros((3, 2, 3)), np.zeros((3, 2, 1))]
    out = tt.tt_round(tt.TensorTrain(z))
    ref = O.tt_round(z)
    assert [c.shape for c in out.cores] == [c.shape for c in ref] == [(1, 2, 1)] * 3
    assert all(not np.any(c) for c in out.cores)
    ranks = [1, 2, 4, 8, 8, 4, 2, 1]
    x = [rng.standard_normal((ranks[k], 2, ranks[k + 1])) for k in range(7)]
    for tol, cap in ((1e-12, 3), (0.3, None), (0.0, 2)):
        out = tt.tt_round(tt.TensorTrain(x), tt.TruncationPolicy(tol, cap))
        ref = O.tt_round(x, tol, cap)
        assert [c.shape for c in out.cores] == [c.shape for c in ref], (tol, cap)
        assert all(a <= b for a, b in zip([c.shape[2] for c in out.cores], ranks[1:]))
        assert rel(O.tt_full(list(out.cores)), O.tt_full(ref)) <= 1e-11
    A = [rng.standard_normal((1, 2, 3, 1))] + [rng.standard_normal((1, 2, 2, 1)) for _ in range(6)]
    with pytest.raises(ShapeMismatchError):
        tt.tt_apply(tt.TTLinearOperator(A), tt.TensorTrain(x))


def _spd_local(rl, R, rr, m, seed, eps=0.5, env_eps=1.0):
    rng = np.random.default_rng(seed)
    gl = rng.standard_normal((R, rl, rl))
    phil = np.einsum("aij,akj->iak", gl, gl) / rl + env_eps * np.eye(rl)[:, None, :]
    gr = rng.standard_normal((R, rr, rr))
    phir = np.einsum("aij,akj->iak", gr, gr) / rr + env_eps * np.eye(rr)[:, None, :]
    G = rng.standard_normal((R, m, m, R)) / R
    A = np.einsum("amnb,apnb->ampb", G, G) + eps * np.einsum("ab,mn->amnb", np.eye(R), np.eye(m))
    rhs = rng.standard_normal((rl, m, rr))
    prev = rng.standard_normal((rl, m, rr)) * 0.1
    from paper_2501_12151_b200 import _native as nat
    return [nat.f64(a) for a in (phil, A, phir, rhs, prev)]


def _local_solve(arrs, rl, R, m, rr, tol, cap, fused):
    from paper_2501_12151_b200 import _native as nat
    phil, A, phir, rhs, prev = arrs
    u = np.empty((rl, m, rr))
    lam, its = ctypes.c_double(), ctypes.c_int()
    nat.call("qtt_local_solve", nat.default_context().handle, nat.dptr(phil), nat.dptr(A), nat.dptr(phir),
             nat.dptr(rhs), nat.dptr(prev), rl, R, m, R, rr, 1, 4096, tol, cap, fused, nat.dptr(u),
             ctypes.byref(lam), ctypes.byref(its))
    return u, lam.value, its.value


@pytest.mark.parametrize("rl,R,rr", [(13, 6, 11), (45, 17, 40)])
def test_cg_odd_leading_width_kernel_vs_oracle(rl, R, rr):
    """Local systems with an odd lk*n (here the 3-component leading core shape, m = 3 and an odd
    rank) cannot use the TMA kernel (16-byte row strides): they run the cp.async persistent CG
    kernel (csrc/cg_fused.cu).  Forced here, against the stepwise path and the oracle's
    restatement of SciPy's cg (amen.py:192-214)."""
    m = 3
    arrs = _spd_local(rl, R, rr, m, seed=rl)
    u1, l1, i1 = _local_solve(arrs, rl, R, m, rr, 1e-6, 400, 1)
    u0, l0, i0 = _local_solve(arrs, rl, R, m, rr, 1e-6, 400, 0)
    assert abs(i0 - i1) <= 1 and rel(u1, u0) <= 1e-9 and abs(l0 - l1) <= 1e-12 * abs(l0)
    phil, A, phir, rhs, prev = arrs
    uo, lo, info = O.solve_local(phil, A, phir, rhs, prev, direct=False, direct_cap=4096, tol=1e-6,
                                 iter_cap=400, sweep=1, k=0)
    assert rel(u1, uo) <= 1e-8 and abs(info["iters"] - i1) <= 1


def test_cg_recurrence_at_the_iteration_cap():
    """the persistent kernel updates q = A z + beta q instead of recomputing q = A p.
    On the real full-rank C3 local system of the committed state fixture (sweep 25, core 15,
    100 x 2 x 98, where the solve runs to the 400-iteration cap), the recurrence must not drift:
    the true residual ||b - A x|| of the fused kernel's solution equals the stepwise path's
    (q = A p every iteration) and the solutions agree to the accuracy two capped runs allow."""
    import os
    from paper_2501_12151_b200 import _native as nat
    from paper_2501_12151_b200 import kernels
    from tests.golden_io import GOLDEN, load_qstep
    fx = load_qstep(os.path.join(GOLDEN, "headline", "c3_step_s25_k15.ref.qstep"))
    x_k, _, _, phil, phir, _, _, psil, psir, _, _, a3, fk = fx["inputs"]
    m = x_k.shape[1]
    A = nat.f64(a3.reshape(a3.shape[0], m, m, a3.shape[2]))
    rhs = nat.f64(kernels.local_rhs(psil[:, :, 0], fk, psir[:, :, 0]))
    arrs = [nat.f64(a) for a in (phil, A, phir, rhs, x_k)]
    rl, R, rr = phil.shape[0], A.shape[0], phir.shape[0]
    phil, A, phir, rhs, prev = arrs
    u1, _, i1 = _local_solve_r(arrs, rl, A.shape[0], m, A.shape[3], rr, 1e-6, 400, 1)
    u0, _, i0 = _local_solve_r(arrs, rl, A.shape[0], m, A.shape[3], rr, 1e-6, 400, 0)
    assert i1 == i0 == 400
    b = np.linalg.norm(rhs)
    r1 = np.linalg.norm(rhs - kernels.local_matvec(phil, A, phir, u1)) / b
    r0 = np.linalg.norm(rhs - kernels.local_matvec(phil, A, phir, u0)) / b
    # measured: 3.17e-6 (fused) vs 3.09e-6 (stepwise) true relative residual after 400 iterations
    # -- two capped runs of the same recurrence in different summation orders; the fused
    # recurrence shows no drift beyond that spread
    assert abs(r1 - r0) <= 0.1 * r0, (r1, r0)
    assert rel(u1, u0) <= 1e-3, rel(u1, u0)


def _local_solve_r(arrs, rl, R0, m, R1, rr, tol, cap, fused):
    from paper_2501_12151_b200 import _native as nat
    phil, A, phir, rhs, prev = arrs
    u = np.empty((rl, m, rr))
    lam, its = ctypes.c_double(), ctypes.c_int()
    nat.call("qtt_local_solve", nat.default_context().handle, nat.dptr(phil), nat.dptr(A), nat.dptr(phir),
             nat.dptr(rhs), nat.dptr(prev), rl, R0, m, R1, rr, 1, 4096, tol, cap, fused, nat.dptr(u),
             ctypes.byref(lam), ctypes.byref(its))
    return u, lam.value, its.value
