"""GPU parity of the interface contractions (K1-K4) against the reference fixtures
and the CPU oracle.  Bar: <= 1e-12 relative (north_star, FP64)."""
import numpy as np
import pytest

from oracle import qtt_oracle as O
from tests.golden_io import load

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def K():
    from paper_2501_12151_b200 import kernels
    return kernels


@pytest.mark.parametrize("fx", ["kernels_bin.npz", "kernels_lead3.npz"])
def test_contractions_vs_reference(K, fx):
    d = load(fx)
    x, z, A, f = d["xk"], d["zk"], d["Ak"], d["fk"]
    assert rel(K.local_matvec(d["phil"], A, d["phir"], x), d["out_local_matvec"]) <= TOL
    assert rel(K.phi_left_step(d["phil"], x, A, x), d["out_phi_left"]) <= TOL
    assert rel(K.phi_right_step(d["phir"], x, A, x), d["out_phi_right"]) <= TOL
    assert rel(K.phi_left_step(d["phizl"], z, A, x), d["out_phiz_left"]) <= TOL
    assert rel(K.phi_right_step(d["phizr"], z, A, x), d["out_phiz_right"]) <= TOL
    assert rel(K.psi_left_step(d["psil"], x, f), d["out_psi_left"]) <= TOL
    assert rel(K.psi_right_step(d["psir"], x, f), d["out_psi_right"]) <= TOL
    assert rel(K.psi_left_step(d["psizl"], z, f), d["out_psiz_left"]) <= TOL
    assert rel(K.local_rhs(d["psil"], f, d["psir"]), d["out_local_rhs"]) <= TOL
    assert rel(K.local_diag(d["phil"], A, d["phir"]), d["out_local_diag"]) <= TOL
    mr = K.mixed_residual(d["psizl"], f, d["psizr"], d["phizl"], A, x, d["phizr"])
    assert rel(mr, d["out_mixed_residual"]) <= 1e-11
    if "out_local_dense" in d:
        assert rel(K.local_dense(d["phil"], A, d["phir"]), d["out_local_dense"]) <= TOL


@pytest.mark.parametrize("r,R,n,m", [(1, 1, 2, 2), (3, 2, 3, 3), (17, 5, 2, 2), (33, 16, 2, 2),
                                     (64, 16, 2, 2), (70, 46, 2, 2), (130, 9, 2, 2)])
def test_contractions_random_shapes(K, r, R, n, m):
    """Ragged/odd shapes (tile edges, rank 1) vs the oracle at config-4-like scales."""
    rng = np.random.default_rng(r * 1000 + R)
    rl, rr = r, max(1, r - 3)
    phil = rng.standard_normal((rl, R, rl))
    phir = rng.standard_normal((rr, R + 1, rr))
    A = rng.standard_normal((R, m, n, R + 1)) / np.sqrt(R)
    x = rng.standard_normal((rl, n, rr))
    assert rel(K.local_matvec(phil, A, phir, x), O.local_matvec(phil, A, phir, x)) <= TOL
    xb = rng.standard_normal((rl, m, rr + 2))
    xk = rng.standard_normal((rl, n, rr))
    assert rel(K.phi_left_step(phil, xb, A, xk), O.env_left(phil, xb, A, xk)) <= TOL
    phi_r = rng.standard_normal((rr + 2, R + 1, rr))
    xb2 = rng.standard_normal((rl + 1, m, rr + 2))
    xk2 = rng.standard_normal((rl, n, rr))
    assert rel(K.phi_right_step(phi_r, xb2, A, xk2), O.env_right(phi_r, xb2, A, xk2)) <= TOL
    if rl * m * rr <= 2048:
        assert rel(K.local_dense(phil, A, phir), O.local_dense(phil, A, phir)) <= TOL
    assert rel(K.local_diag(phil, A, phir), O.local_diag(phil, A, phir)) <= TOL


def test_c4_shapes_r128(K):
    """Config-4 interior core at r=128, R=16 (BASELINE.json configs[3])."""
    rng = np.random.default_rng(1)
    r, R = 128, 16
    phil = rng.standard_normal((r, R, r)) / r
    phir = rng.standard_normal((r, R, r)) / r
    A = rng.standard_normal((R, 2, 2, R)) / np.sqrt(r)
    x = rng.standard_normal((r, 2, r)) / np.sqrt(r)
    assert rel(K.local_matvec(phil, A, phir, x), O.local_matvec(phil, A, phir, x)) <= TOL
    assert rel(K.phi_left_step(phil, x, A, x), O.env_left(phil, x, A, x)) <= TOL
    assert rel(K.phi_right_step(phir, x, A, x), O.env_right(phir, x, A, x)) <= TOL


def test_shape_errors(K):
    from paper_2501_12151_b200.errors import ShapeMismatchError
    with pytest.raises(ShapeMismatchError):
        K.local_matvec(np.ones((2, 3, 2)), np.ones((3, 2, 2, 3)), np.ones((2, 3, 2)), np.ones((2, 3, 2)))
