"""3D Q1 elasticity assembly (paper_2501_12151_b200.assembly3d) against
an independent element-loop scipy.sparse oracle (oracle/elasticity_fem.py), following the
reference's own checks of its 2D assembly: dense scatter vs the QTT operator
(/root/reference/pkg/tests/test_elasticity.py:414-432) and the rigid-body null space
(test_elasticity.py:226-239), plus the clamp, SPD-ness, body and patch loads and the
two-layer material with a cut element (config C5)."""
import numpy as np
import pytest

from oracle import elasticity_fem as F
from oracle import qtt_oracle as O
from paper_2501_12151_b200.assembly3d import assemble_cube, stiffness_qtt

LAYERS = (0.5, 1.0, 10.0)  # C5: E = 1 below z = 0.5, 10 above


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("L,layers", [(2, None), (3, None), (2, LAYERS), (3, LAYERS)])
def test_stiffness_vs_element_loop(L, layers):
    """Kronecker/QTT stiffness == element-loop stiffness; at L = 2, 3 the z = 0.5 interface
    cuts an element (h = 1/3, 1/7), integrated exactly on both sides."""
    K = F.stiffness(L, layers=layers).toarray()
    Kq = O.op_full(stiffness_qtt(L, layers=layers))
    assert rel(Kq, K) <= 1e-13
    assert np.abs(Kq - Kq.T).max() <= 1e-13 * np.abs(Kq).max()


@pytest.mark.parametrize("layers", [None, LAYERS])
def test_rigid_body_null_space(layers):
    L = 3
    Kq = O.op_full(stiffness_qtt(L, layers=layers))
    R = F.rigid_body_modes(L)
    for r in R:
        assert np.linalg.norm(Kq @ r) <= 1e-12 * np.linalg.norm(Kq) * np.linalg.norm(r)
    # and nothing else: exactly six (near-)zero eigenvalues of the unclamped stiffness
    ev = np.linalg.eigvalsh(Kq)
    assert (ev < 1e-10 * ev[-1]).sum() == 6


@pytest.mark.parametrize("L,layers,load", [(2, None, "body"), (3, None, "body"), (2, LAYERS, "patch"),
                                           (3, LAYERS, "patch"), (3, None, "patch")])
def test_clamped_system_vs_element_loop(L, layers, load):
    """assemble_cube (clamp P K P + (I - P), scaling, load) == the oracle's clamped system."""
    prob = assemble_cube(L, layers=layers, load=load, rounding="host")
    K = F.stiffness(L, layers=layers)
    f = F.body_load(L) if load == "body" else F.patch_load(L)
    A, rhs, s = F.clamped_system(K, f, L)
    Aq = O.op_full(prob.op)
    assert abs(prob.scale - s) <= 1e-13 * s
    assert rel(Aq, A.toarray()) <= 1e-13
    assert rel(O.tt_full(prob.rhs), rhs) <= 1e-13
    ev = np.linalg.eigvalsh(Aq)
    assert ev[0] > 0, "clamped operator must be SPD"


def test_patch_load_total_force():
    """The patch traction integrates to traction x patch area (0.5 x 0.5) in every config."""
    for L in (2, 3, 4):
        f = F.patch_load(L).reshape(3, -1)
        assert abs(f[2].sum() + 0.25) <= 1e-14 and abs(f[0].sum()) == 0.0


def test_body_load_total_force():
    for L in (2, 3):
        f = F.body_load(L).reshape(3, -1)
        assert abs(f[2].sum() + 1.0) <= 1e-13


def test_operator_ranks_c1():
    """MPO ranks of the solver operator at C1 (L = 5; 45)."""
    prob = assemble_cube(5, rounding="host")
    assert max(prob.op_ranks) == 45
    assert prob.dims == (3,) + (2,) * 15
