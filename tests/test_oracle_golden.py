"""Pin the CPU oracle (oracle/qtt_oracle.py) against the reference's frozen outputs.

CPU-only.  The fixtures come from running the real reference (tests/golden/make_golden.py).
"""
import numpy as np
import pytest

from oracle import qtt_oracle as O
from tests.golden_io import AMEN_CASES, amen_config, load, train


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("fx", ["kernels_bin.npz", "kernels_lead3.npz"])
def test_interface_contractions(fx):
    d = load(fx)
    x, z, A, f = d["xk"], d["zk"], d["Ak"], d["fk"]
    assert rel(O.local_matvec(d["phil"], A, d["phir"], x), d["out_local_matvec"]) <= 1e-13
    assert rel(O.env_left(d["phil"], x, A, x), d["out_phi_left"]) <= 1e-13
    assert rel(O.env_right(d["phir"], x, A, x), d["out_phi_right"]) <= 1e-13
    assert rel(O.env_left(d["phizl"], z, A, x), d["out_phiz_left"]) <= 1e-13
    assert rel(O.env_right(d["phizr"], z, A, x), d["out_phiz_right"]) <= 1e-13
    assert rel(O.rhs_env_left(d["psil"], x, f), d["out_psi_left"]) <= 1e-13
    assert rel(O.rhs_env_right(d["psir"], x, f), d["out_psi_right"]) <= 1e-13
    assert rel(O.rhs_env_left(d["psizl"], z, f), d["out_psiz_left"]) <= 1e-13
    assert rel(O.local_rhs(d["psil"], f, d["psir"]), d["out_local_rhs"]) <= 1e-13
    assert rel(O.local_diag(d["phil"], A, d["phir"]), d["out_local_diag"]) <= 1e-13
    mr = O.mixed_residual(d["psizl"], f, d["psizr"], d["phizl"], A, x, d["phizr"])
    assert rel(mr, d["out_mixed_residual"]) <= 1e-12
    if "out_local_dense" in d:
        assert rel(O.local_dense(d["phil"], A, d["phir"]), d["out_local_dense"]) <= 1e-13


def test_truncated_factor_and_rank_rule():
    d = load("factor.npz")
    for i in range(int(d["tf_count"])):
        rel_tol, cap, dabs = d[f"tf{i}_pol"]
        q, w = O.truncated_factor(d[f"tf{i}_mat"], rel_tol, None if cap < 0 else int(cap),
                                  None if dabs < 0 else dabs)
        assert q.shape[1] == int(d[f"tf{i}_rank"]), i
        assert np.linalg.norm(q @ w - d[f"tf{i}_qw"]) <= 1e-12 * max(1.0, np.linalg.norm(d[f"tf{i}_qw"]))
    for j in range(int(d["rr_count"])):
        assert O.rank_for_tolerance(d[f"rr{j}_s"], float(d[f"rr{j}_delta"])) == int(d[f"rr{j}_r"])


def test_tt_ops():
    d = load("tt_ops.npz")
    v, w, A = train(d, "v"), train(d, "w"), train(d, "A")
    orth = O.orthogonalize_rl(v)
    ref = train(d, "v_orth")
    assert [c.shape for c in orth] == [c.shape for c in ref]
    assert rel(O.tt_full(orth), O.tt_full(ref)) <= 1e-13
    assert abs(O.tt_norm(v) - float(d["v_norm"])) <= 1e-13 * float(d["v_norm"])
    assert abs(O.tt_dot(v, w) - float(d["vw_dot"])) <= 1e-12 * abs(float(d["vw_dot"]))
    s = O.tt_add(v, w)
    for j in range(4):
        tol, cap = d[f"round{j}_pol"]
        out = O.tt_round(s, tol, None if cap < 0 else int(cap))
        refj = train(d, f"round{j}")
        assert [c.shape for c in out] == [c.shape for c in refj], j
        assert rel(O.tt_full(out), O.tt_full(refj)) <= 1e-12
    dbl = O.tt_round(O.tt_add(v, v))
    assert [c.shape for c in dbl] == [c.shape for c in train(d, "round_double")]
    av = O.tt_apply(A, v)
    for c, r in zip(av, train(d, "Av")):
        assert c.shape == r.shape and rel(c, r) <= 1e-15
    avr = O.tt_round(av, 1e-8)
    assert [c.shape for c in avr] == [c.shape for c in train(d, "Av_round")]
    assert abs(O.residual_norm(A, v, w) - float(d["resid_none"])) <= 1e-12 * float(d["resid_none"])
    assert abs(O.residual_norm(A, v, w, (1e-9, None)) - float(d["resid_round"])) <= 1e-9 * float(d["resid_round"])


def test_solve_local():
    d = load("solve_local.npz")
    u, lam, _ = O.solve_local(d["phil"], d["Ak"], d["phir"], d["rhs"], d["prev"], direct=True,
                              direct_cap=4096, tol=1e-8, iter_cap=400, sweep=1, k=2)
    assert rel(u, d["direct_u"]) <= 1e-12
    assert abs(lam - float(d["direct_lam"])) <= 1e-12 * float(d["direct_lam"])
    for tol in (1e-8, 1e-4):
        u, lam, _ = O.solve_local(d["phil"], d["Ak"], d["phir"], d["rhs"], d["prev"], direct=False,
                                  direct_cap=4096, tol=tol, iter_cap=400, sweep=1, k=2)
        assert rel(u, d[f"iter_u_{tol:g}"]) <= 1e-10
        assert abs(lam - float(d[f"iter_lam_{tol:g}"])) <= 1e-12 * abs(float(d[f"iter_lam_{tol:g}"]))


def check_amen_parity(d, rep, x_full):
    """Trajectory parity against the reference fixture (shared with the GPU tests).

    Converged reference runs: same convergence, same sweep count and rank history,
    certified residual <= tol and the decompressed field within 10 x tol (north star).
    Rank-limited (non-converged) runs are chaotic in floating point -- the reference's
    own 1e-15-perturbed ensemble spreads by tens of percent (tests/golden/make_golden.py)
    -- so the final residual must fall inside that band widened by 10%.
    """
    tol = float(d["cfg_residual_tol"])
    lo, hi = (float(v) for v in d["band_final"])
    final = rep["final_relative_residual"]
    if bool(d["band_converged_all"]):
        assert rep["converged"]
        assert final <= tol
        assert rep["sweeps_used"] == int(d["rep_sweeps_used"])
        hist = np.array(rep["rank_profile_history"]).reshape(d["rep_rank_hist"].shape)
        assert np.array_equal(hist, d["rep_rank_hist"])
        xr = O.tt_full(train(d, "x"))
        assert np.linalg.norm(x_full - xr) <= 10 * tol * np.linalg.norm(xr)
    else:
        assert 0.9 * lo <= final <= 1.1 * hi, (final, lo, hi)


@pytest.mark.parametrize("case", AMEN_CASES)
def test_amen_trajectory(case):
    d = load(case)
    x0 = train(d, "x0") if "x0__n" in d else None
    x, rep = O.amen_solve(train(d, "A"), train(d, "f"), x0, amen_config(d))
    check_amen_parity(d, rep, O.tt_full(x))


def test_op_round_oracle_vs_reference():
    """The oracle's tt_round over fused (m*n) modes reproduces the reference's tt_op_round."""
    d = load("op_round.npz")
    for name, (tol, cap) in (("AA", (1e-10, None)), ("B", (1e-2, 3))):
        A = train(d, name)
        fused = [c.reshape(c.shape[0], c.shape[1] * c.shape[2], c.shape[3]) for c in A]
        out = O.tt_round(fused, tol, cap)
        ref = train(d, f"{name}_round")
        assert [c.shape[0] for c in out] == [c.shape[0] for c in ref]
        outc = [c.reshape(r.shape) for c, r in zip(out, ref)]
        assert rel(O.op_full(outc), O.op_full(ref)) <= 1e-12
