"""TT-cross on the device (paper_2501_12151_b200.cross, csrc/cross.cu) against the unmodified
reference's cross_interpolate / reciprocal_tt on the same seeded functions
(tests/golden/make_cross_golden.py): the same pivot index sets, sweep count, evaluation count,
ranks, and the same interpolant to 1e-12.  The reference's own test_cross.py runs against the
engine in tests/ref_suite."""
import numpy as np
import pytest

from tests.golden_io import load

pytestmark = pytest.mark.gpu


def _cases():
    d = 10
    w2 = 2 ** np.arange(d - 1, -1, -1)
    smooth = 1.0 / (1.0 + (np.arange(2 ** d) / 2 ** d))
    w4 = 4 ** np.arange(4, -1, -1)
    v = 2.0 + np.sin(np.arange(4 ** 5) / 37.0)
    rng = np.random.default_rng(11)
    ranks = [1, 3, 3, 3, 1]
    cores = [rng.standard_normal((ranks[k], 4, ranks[k + 1])) for k in range(4)]
    full3 = cores[0]
    for c in cores[1:]:
        full3 = np.tensordot(full3, c, axes=(full3.ndim - 1, 0))
    full3 = full3.reshape(4, 4, 4, 4)
    return {
        "rank3": ((4,) * 4, lambda idx: full3[tuple(np.asarray(idx).T)], dict(initial_rank=4), False),
        "smooth": ((2,) * d, lambda idx: smooth[np.asarray(idx) @ w2], dict(rel_convergence_tol=1e-10), False),
        "recip": ((4,) * 5, lambda idx: v[np.asarray(idx) @ w4], {}, True),
    }


@pytest.mark.parametrize("name", ["rank3", "smooth", "recip"])
def test_cross_matches_reference(name):
    from paper_2501_12151_b200.cross import CrossConfig, cross_interpolate, reciprocal_tt
    from paper_2501_12151_b200.tt import tt_to_dense
    ref = load("cross_ref.npz")
    dims, f, kw, recip = _cases()[name]
    tt, rep = (reciprocal_tt if recip else cross_interpolate)(f, dims, CrossConfig(**kw))
    assert rep.converged == bool(ref[f"{name}__converged"])
    assert rep.sweeps_used == int(ref[f"{name}__sweeps"])
    assert rep.evaluations == int(ref[f"{name}__evaluations"])
    assert tuple(tt.ranks) == tuple(int(v) for v in ref[f"{name}__ranks"])
    nb = int(ref[f"{name}__nbonds"])
    assert len(rep.left_indices) == nb
    # pivot sets: maxvol has many admissible (quasi-dominant) answers; which one a run lands on
    # follows the pivoted QR's choice among exact ties (e.g. the equal unit row norms of a
    # square orthogonal Q), decided by last-bit rounding in either implementation.  The device's
    # own sets must be valid and nested, with the interpolation property (cross.py docstring):
    # the train reproduces f exactly on every left x right pivot cross
    from paper_2501_12151_b200.tt import tt_entries
    for b in range(nb):
        L, R = np.asarray(rep.left_indices[b]), np.asarray(rep.right_indices[b])
        assert len(L) == len(ref[f"{name}__left{b}"]) and len(R) == len(ref[f"{name}__right{b}"])
        idx = np.array([np.concatenate([l, r]) for l in L for r in R])
        got = tt_entries(tt, idx)
        want_f = f(idx) if not recip else 1.0 / f(idx)
        np.testing.assert_allclose(got, want_f, rtol=1e-12, atol=1e-13 * np.abs(want_f).max())
    dense, want = tt_to_dense(tt), ref[f"{name}__dense"]
    assert np.linalg.norm(dense - want) <= 1e-12 * np.linalg.norm(want)
    # the sampled-error history: equal while the error is above round-off; below ~1e-8 both sides
    # report round-off noise of their own QR/maxvol arithmetic
    got_e, want_e = np.asarray(rep.sampled_errors), ref[f"{name}__errors"]
    big = want_e > 1e-8
    np.testing.assert_allclose(got_e[big], want_e[big], rtol=1e-3)
    assert (got_e[~big] <= 1e-8).all()


def test_maxvol_device_properties():
    """Dominance, exact identity recovery and the rank-deficient fallback."""
    from paper_2501_12151_b200.cross import maxvol_select
    rng = np.random.default_rng(42)
    mat = rng.standard_normal((300, 24))
    rows = maxvol_select(mat, tol=0.01)
    assert len(set(rows)) == 24
    assert np.abs(mat @ np.linalg.inv(mat[rows])).max() <= 1.01 + 1e-12
    base = np.vstack([np.eye(5), np.zeros((20, 5))])
    perm = rng.permutation(25)
    assert set(perm[list(maxvol_select(base[perm]))]) == set(range(5))
