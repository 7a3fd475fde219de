"""Generate golden fixtures by running the REAL reference (``ttfem``) in the build
container.  Run from the repo root:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference is pure Python and does not exist on the GPU box, so its outputs are
frozen here as small ``.npz`` files that travel with the repo.  The reference's
``_ALLOWED_MODES`` (tt.py:61) is widened at runtime (no file edit) so it accepts the
3-component leading core of the 3D problems.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import ttfem.tt as rtt  # noqa: E402
import ttfem.amen as ram  # noqa: E402

rtt._ALLOWED_MODES = (2, 3, 4, 8, 9)

from paper_2501_12151_b200.assembly3d import assemble_cube  # noqa: E402


def put_train(d, name, cores):
    d[f"{name}__n"] = np.array(len(cores))
    for k, c in enumerate(cores):
        d[f"{name}__{k}"] = np.ascontiguousarray(c, dtype=np.float64)


def rand_train(rng, dims, ranks, scale=1.0):
    full = [1] + list(ranks) + [1]
    return [scale * rng.standard_normal((full[k], dims[k], full[k + 1])) for k in range(len(dims))]


def rand_op(rng, dims, ranks, scale=1.0):
    full = [1] + list(ranks) + [1]
    return [scale * rng.standard_normal((full[k], dims[k], dims[k], full[k + 1])) for k in range(len(dims))]


def kernels_case(seed, dims, r, R, rz):
    """Interface contractions on one interior core, environments built by the
    reference's own env functions (Appendix B of SURVEY.md)."""
    rng = np.random.default_rng(seed)
    K = len(dims)
    x = rand_train(rng, dims, [r] * (K - 1), 1.0 / np.sqrt(r))
    z = rand_train(rng, dims, [rz] * (K - 1), 1.0 / np.sqrt(rz))
    A = rand_op(rng, dims, [R] * (K - 1), 1.0 / np.sqrt(R))
    f = rand_train(rng, dims, [3] * (K - 1))
    k = K // 2
    one3, one2 = np.ones((1, 1, 1)), np.ones((1, 1))
    phil, phizl, psil, psizl = one3, one3, one2, one2
    for j in range(k):
        phil = ram._phi_left_step(phil, x[j], A[j], x[j])
        phizl = ram._phi_left_step(phizl, z[j], A[j], x[j])
        psil = ram._psi_left_step(psil, x[j], f[j])
        psizl = ram._psi_left_step(psizl, z[j], f[j])
    phir, phizr, psir, psizr = one3, one3, one2, one2
    for j in range(K - 1, k, -1):
        phir = ram._phi_right_step(phir, x[j], A[j], x[j])
        phizr = ram._phi_right_step(phizr, z[j], A[j], x[j])
        psir = ram._psi_right_step(psir, x[j], f[j])
        psizr = ram._psi_right_step(psizr, z[j], f[j])
    d = {}
    d.update(xk=x[k], zk=z[k], Ak=A[k], fk=f[k], phil=phil, phir=phir, phizl=phizl,
             phizr=phizr, psil=psil, psir=psir, psizl=psizl, psizr=psizr)
    d["out_local_matvec"] = ram._local_matvec(phil, A[k], phir, x[k])
    d["out_phi_left"] = ram._phi_left_step(phil, x[k], A[k], x[k])
    d["out_phi_right"] = ram._phi_right_step(phir, x[k], A[k], x[k])
    d["out_phiz_left"] = ram._phi_left_step(phizl, z[k], A[k], x[k])
    d["out_phiz_right"] = ram._phi_right_step(phizr, z[k], A[k], x[k])
    d["out_psi_left"] = ram._psi_left_step(psil, x[k], f[k])
    d["out_psi_right"] = ram._psi_right_step(psir, x[k], f[k])
    d["out_psiz_left"] = ram._psi_left_step(psizl, z[k], f[k])
    d["out_local_rhs"] = ram._local_rhs(psil, f[k], psir)
    d["out_local_diag"] = ram._local_diag(phil, A[k], phir)
    d["out_mixed_residual"] = ram._mixed_residual(psizl, f[k], psizr, phizl, A[k], x[k], phizr)
    dim = phil.shape[0] * dims[k] * phir.shape[0]
    if dim <= 1500:
        d["out_local_dense"] = ram._local_dense(phil, A[k], phir)
    return d


def factor_cases():
    d = {}
    rng = np.random.default_rng(5)
    mats = []
    for (m, n, decay) in [(24, 12, 0.5), (40, 20, 0.3), (16, 16, 0.9), (30, 7, 1e-3), (9, 30, 0.6)]:
        u, _ = np.linalg.qr(rng.standard_normal((m, min(m, n))))
        v, _ = np.linalg.qr(rng.standard_normal((n, min(m, n))))
        s = decay ** np.arange(min(m, n))
        mats.append(u @ np.diag(s) @ v.T)
    mats.append(np.zeros((6, 4)))
    mats.append(rng.standard_normal((12, 5)))
    pols = [(1e-10, 80, None), (1e-3, None, None), (1e-2, 4, None), (0.0, None, None),
            (1e-10, 80, 1e-4), (0.5, None, 1e-9)]
    i = 0
    for mi, mat in enumerate(mats):
        for (rel, cap, dabs) in pols:
            q, w = ram._truncated_factor(mat, rtt.TruncationPolicy(rel, cap), dabs)
            d[f"tf{i}_mat"] = mat
            d[f"tf{i}_pol"] = np.array([rel, -1 if cap is None else cap, -1 if dabs is None else dabs])
            d[f"tf{i}_rank"] = np.array(q.shape[1])
            d[f"tf{i}_qw"] = q @ w
            d[f"tf{i}_s"] = np.linalg.svd(mat, compute_uv=False)
            i += 1
    d["tf_count"] = np.array(i)
    # rank rule edge cases
    rr = []
    for s, delta in [([3.0, 2.0, 1.0], 0.0), ([3.0, 2.0, 1.0], 1.0), ([3.0, 2.0, 1.0], 2.2361),
                     ([3.0, 2.0, 1.0], 2.23607), ([1.0], 5.0), ([], 1.0), ([1e-300, 1e-300], 0.0),
                     ([5.0, 0.0, 0.0], 0.0)]:
        rr.append((np.array(s, dtype=np.float64), delta, rtt._rank_for_tolerance(np.array(s, dtype=np.float64), delta)))
    for j, (s, delta, r) in enumerate(rr):
        d[f"rr{j}_s"] = s
        d[f"rr{j}_delta"] = np.array(delta)
        d[f"rr{j}_r"] = np.array(r)
    d["rr_count"] = np.array(len(rr))
    return d


def tt_cases():
    d = {}
    rng = np.random.default_rng(11)
    dims = (3, 2, 2, 2, 2, 2, 2, 2)
    v = rtt.TensorTrain(rand_train(rng, dims, [2, 4, 6, 6, 6, 4, 2]))
    put_train(d, "v", v.cores)
    orth = rtt._orthogonalize_rl(list(v.cores))
    put_train(d, "v_orth", orth)
    d["v_norm"] = np.array(rtt.tt_norm(v))
    w = rtt.TensorTrain(rand_train(rng, dims, [3, 3, 3, 3, 3, 3, 3]))
    put_train(d, "w", w.cores)
    d["vw_dot"] = np.array(rtt.tt_dot(v, w))
    s = rtt.tt_add(v, w)
    for j, (tol, cap) in enumerate([(1e-12, None), (1e-2, None), (0.0, 3), (0.3, None)]):
        out = rtt.tt_round(s, rtt.TruncationPolicy(tol, cap))
        put_train(d, f"round{j}", out.cores)
        d[f"round{j}_pol"] = np.array([tol, -1 if cap is None else cap])
    dbl = rtt.tt_round(rtt.tt_add(v, v))
    put_train(d, "round_double", dbl.cores)
    A = rtt.TTLinearOperator(rand_op(rng, dims, [3, 4, 4, 4, 4, 4, 3], 0.5))
    put_train(d, "A", A.cores)
    Av = rtt.tt_apply(A, v, policy=None)
    put_train(d, "Av", Av.cores)
    Avr = rtt.tt_apply(A, v, rtt.TruncationPolicy(1e-8))
    put_train(d, "Av_round", Avr.cores)
    d["resid_none"] = np.array(ram.residual_norm(A, v, w))
    d["resid_round"] = np.array(ram.residual_norm(A, v, w, rtt.TruncationPolicy(1e-9)))
    return d


def solve_local_cases():
    d = {}
    rng = np.random.default_rng(13)
    # SPD local system: build envs from an SPD operator G^T G + I
    dims = (3, 2, 2, 2, 2, 2)
    K = len(dims)
    g = rtt.TTLinearOperator(rand_op(rng, dims, [2] * (K - 1), 0.5))
    A = rtt.tt_op_add(rtt.tt_op_compose(rtt.tt_op_transpose(g), g), rtt.tt_identity(dims))
    x = rtt._orthogonalize_rl(rand_train(rng, dims, [3, 5, 6, 5, 2]))
    f = rand_train(rng, dims, [2] * (K - 1))
    k = 2
    one3, one2 = np.ones((1, 1, 1)), np.ones((1, 1))
    # left-orthogonalize cores < k
    cores = list(x)
    for j in range(k):
        r0, n, r1 = cores[j].shape
        q, r = np.linalg.qr(cores[j].reshape(r0 * n, r1))
        cores[j] = q.reshape(r0, n, q.shape[1])
        cores[j + 1] = np.einsum("ab,bnc->anc", r, cores[j + 1])
    # right-orthogonalize cores > k
    for j in range(K - 1, k, -1):
        r0, n, r1 = cores[j].shape
        q, r = np.linalg.qr(cores[j].reshape(r0, n * r1).T)
        cores[j] = q.T.reshape(q.shape[1], n, r1)
        cores[j - 1] = np.einsum("anb,bc->anc", cores[j - 1], r.T)
    phil, psil = one3, one2
    for j in range(k):
        phil = ram._phi_left_step(phil, cores[j], A.cores[j], cores[j])
        psil = ram._psi_left_step(psil, cores[j], f[j])
    phir, psir = one3, one2
    for j in range(K - 1, k, -1):
        phir = ram._phi_right_step(phir, cores[j], A.cores[j], cores[j])
        psir = ram._psi_right_step(psir, cores[j], f[j])
    rhs = ram._local_rhs(psil, f[k], psir)
    d.update(phil=phil, phir=phir, Ak=A.cores[k], rhs=rhs, prev=cores[k])
    u, lam = ram._solve_local(phil, A.cores[k], phir, rhs, cores[k], ram.AmenConfig(), 1, k)
    d["direct_u"], d["direct_lam"] = u, np.array(lam)
    for tol in (1e-8, 1e-4):
        cfg = ram.AmenConfig(local_solver="iterative", residual_tol=tol)
        u, lam = ram._solve_local(phil, A.cores[k], phir, rhs, cores[k], cfg, 1, k)
        d[f"iter_u_{tol:g}"], d[f"iter_lam_{tol:g}"] = u, np.array(lam)
    return d


def amen_case(name, A, f, x0, cfg_kwargs):
    cfg = ram.AmenConfig(**cfg_kwargs)
    At = rtt.TTLinearOperator(A)
    ft = rtt.TensorTrain(f)
    x0t = None if x0 is None else rtt.TensorTrain(x0)
    x, rep = ram.amen_solve(At, ft, x0=x0t, config=cfg)
    d = {}
    put_train(d, "A", A)
    put_train(d, "f", f)
    if x0 is not None:
        put_train(d, "x0", x0)
    put_train(d, "x", x.cores)
    d["cfg_residual_tol"] = np.array(cfg.residual_tol)
    d["cfg_max_sweeps"] = np.array(cfg.max_sweeps)
    d["cfg_enrichment_rank"] = np.array(cfg.enrichment_rank)
    d["cfg_local_solver"] = np.array(cfg.local_solver)
    d["cfg_direct_dim_cap"] = np.array(cfg.direct_dim_cap)
    d["cfg_local_iter_cap"] = np.array(cfg.local_iter_cap)
    d["cfg_rounding"] = np.array([cfg.rounding.rel_tolerance,
                                  -1 if cfg.rounding.max_rank is None else cfg.rounding.max_rank])
    d["cfg_seed"] = np.array(cfg.seed)
    d["cfg_stagnation_strikes"] = np.array(cfg.stagnation_strikes)
    d["rep_converged"] = np.array(rep.converged)
    d["rep_sweeps_used"] = np.array(rep.sweeps_used)
    d["rep_final"] = np.array(rep.final_relative_residual)
    d["rep_res_hist"] = np.array(rep.residual_history)
    width = max(len(r) for r in rep.rank_profile_history) if rep.rank_profile_history else 0
    d["rep_rank_hist"] = np.array([list(r) for r in rep.rank_profile_history]).reshape(-1, width)
    # The sweep trajectory is sensitive to round-off: lam_max (amen.py:190,330-337)
    # is basis dependent and rank-limited runs are chaotic.  Record the reference's
    # own spread under 1e-15 relative perturbations of x0 (or f when x0 is None);
    # parity tests accept results inside this band (+-10%).
    finals, sweeps = [rep.final_relative_residual], [rep.sweeps_used]
    for s in range(ENSEMBLE):
        prng = np.random.default_rng(1000 + s)
        if x0 is not None:
            x0p = rtt.TensorTrain([c * (1 + 1e-15 * prng.standard_normal(c.shape)) for c in x0])
            fp = ft
        else:
            x0p = None
            fp = rtt.TensorTrain([c * (1 + 1e-15 * prng.standard_normal(c.shape)) for c in f])
        _, rp = ram.amen_solve(At, fp, x0=x0p, config=cfg)
        finals.append(rp.final_relative_residual)
        sweeps.append(rp.sweeps_used)
    d["band_final"] = np.array([min(finals), max(finals)])
    d["band_sweeps"] = np.array([min(sweeps), max(sweeps)])
    d["band_converged_all"] = np.array(all(v <= cfg.residual_tol for v in finals))
    np.savez_compressed(os.path.join(HERE, f"amen_{name}.npz"), **d)
    print(name, rep.converged, rep.sweeps_used, rep.final_relative_residual, x.ranks,
          "band", d["band_final"], d["band_sweeps"])


ENSEMBLE = 8


def x0_rank2(dims, seed=0):
    """rank-2 TT, N(0,1) cores from default_rng(seed), k = 0..K-1."""
    rng = np.random.default_rng(seed)
    K = len(dims)
    return [rng.standard_normal((1 if k == 0 else 2, dims[k], 1 if k == K - 1 else 2)) for k in range(K)]


def spd_op(dims, seed):
    rng = np.random.default_rng(seed)
    g = rtt.TTLinearOperator(rand_op(rng, dims, [2] * (len(dims) - 1), 0.4))
    return list(rtt.tt_op_add(rtt.tt_op_compose(rtt.tt_op_transpose(g), g), rtt.tt_identity(dims)).cores)


def c4_cases():
    """Config 4 at reduced size through the reference's own primitives: the matvec sweep
    (right-env pre-pass, then _local_matvec + _phi_left_step per core) and
    tt_round(tt_apply(A, x, None), TruncationPolicy(1e-8)) (tt.py:409, 434)."""
    from paper_2501_12151_b200.configs import c4_problem
    d = {}
    for tag, (r, dd, R) in {"a": (6, 10, 4), "b": (16, 12, 16)}.items():
        op, x = c4_problem(r, d=dd, R=R, seed=1)
        K = len(op)
        right = [None] * (K + 1)
        right[K] = np.ones((1, 1, 1))
        for k in range(K - 1, 0, -1):
            right[k] = ram._phi_right_step(right[k + 1], x[k], op[k], x[k])
        left = np.ones((1, 1, 1))
        ys = []
        for k in range(K):
            ys.append(ram._local_matvec(left, op[k], right[k + 1], x[k]))
            if k + 1 < K:
                left = ram._phi_left_step(left, x[k], op[k], x[k])
        put_train(d, f"{tag}_A", op)
        put_train(d, f"{tag}_x", x)
        put_train(d, f"{tag}_y", ys)
        y = rtt.tt_apply(rtt.TTLinearOperator(op), rtt.TensorTrain(x), None)
        yr = rtt.tt_round(y, rtt.TruncationPolicy(1e-8))
        if tag == "a":  # (the rank-R*r product train is large; one small case is enough)
            put_train(d, f"{tag}_apply", list(y.cores))
        put_train(d, f"{tag}_round", list(yr.cores))
        d[f"{tag}_round_norm"] = np.array(rtt.tt_norm(yr))
    return d


def qtt1_cases():
    """Reference QTT1 containers (serialize.py:33-49) of a small vector and operator."""
    import ttfem.serialize as rser
    rng = np.random.default_rng(5)
    v = rtt.TensorTrain(rand_train(rng, (3, 2, 2, 2), [2, 3, 2]))
    a = rtt.TTLinearOperator(rand_op(rng, (3, 2, 2), [2, 3]))
    rser.save_tt(v, os.path.join(HERE, "vec.qtt1"))
    rser.save_tt(a, os.path.join(HERE, "op.qtt1"))


def op_round_cases():
    """tt_op_round (tt.py:506-531) of an operator whose ranks double (A + A, A = the L=2 cube
    stiffness of this repo's assembly) and of a random operator, as the reference computes it."""
    d = {}
    A = rtt.TTLinearOperator(assemble_cube(2).op)
    AA = rtt.tt_op_add(A, A)
    put_train(d, "AA", list(AA.cores))
    put_train(d, "AA_round", list(rtt.tt_op_round(AA, rtt.TruncationPolicy(1e-10)).cores))
    rng = np.random.default_rng(21)
    B = rtt.TTLinearOperator(rand_op(rng, (2, 2, 2, 2, 2), [4, 6, 6, 4], 0.5))
    put_train(d, "B", list(B.cores))
    put_train(d, "B_round", list(rtt.tt_op_round(B, rtt.TruncationPolicy(1e-2, 3)).cores))
    np.savez_compressed(os.path.join(HERE, "op_round.npz"), **d)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "opround":
        op_round_cases()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "qtt1":
        qtt1_cases()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "c4":  # regenerate only the config-4 fixture
        np.savez_compressed(os.path.join(HERE, "c4_small.npz"), **c4_cases())
        return
    np.savez_compressed(os.path.join(HERE, "c4_small.npz"), **c4_cases())
    qtt1_cases()
    op_round_cases()
    np.savez_compressed(os.path.join(HERE, "kernels_bin.npz"), **kernels_case(1, (2,) * 8, 12, 6, 4))
    np.savez_compressed(os.path.join(HERE, "kernels_lead3.npz"), **kernels_case(2, (3,) + (2,) * 7, 10, 7, 4))
    np.savez_compressed(os.path.join(HERE, "factor.npz"), **factor_cases())
    np.savez_compressed(os.path.join(HERE, "tt_ops.npz"), **tt_cases())
    np.savez_compressed(os.path.join(HERE, "solve_local.npz"), **solve_local_cases())

    # amen: reference test-style SPD systems
    dims = (4, 4, 4)
    rng = np.random.default_rng(12)
    f = rand_train(rng, dims, [3, 3])
    amen_case("spd444", spd_op(dims, 11), f, None, {})
    amen_case("spd444_iter", spd_op(dims, 31), f, None, {"local_solver": "iterative"})
    # 3D elasticity (this repo's assembly), settings of config C1 at small L
    for L, maxr, extra in [(2, 32, {}), (3, 8, {}), (3, 16, {"max_sweeps": 12}),
                           (2, 32, {"local_solver": "iterative", "residual_tol": 1e-6})]:
        prob = assemble_cube(L)
        x0 = x0_rank2(prob.dims, 0)
        kw = {"residual_tol": 1e-6, "rounding": rtt.TruncationPolicy(1e-6, maxr), "seed": 2024}
        kw.update(extra)
        tag = f"cube_L{L}_r{maxr}" + ("_iter" if extra.get("local_solver") == "iterative" else "") + \
              (f"_s{extra['max_sweeps']}" if "max_sweeps" in extra else "")
        amen_case(tag, prob.op, prob.rhs, x0, kw)


if __name__ == "__main__":
    main()
