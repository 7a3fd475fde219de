"""GPU end-to-end parity of amen_solve against the reference's own trajectories."""
import numpy as np
import pytest

from oracle import qtt_oracle as O
from tests.golden_io import AMEN_CASES, amen_config, load, train
from tests.test_oracle_golden import check_amen_parity

pytestmark = pytest.mark.gpu


def to_config(d):
    from paper_2501_12151_b200.amen import AmenConfig
    from paper_2501_12151_b200.tt import TruncationPolicy
    c = amen_config(d)
    rel, cap = c.pop("rounding")
    return AmenConfig(rounding=TruncationPolicy(rel, cap), **c)


@pytest.mark.parametrize("case", AMEN_CASES)
def test_amen_vs_reference(case):
    from paper_2501_12151_b200.amen import amen_solve
    from paper_2501_12151_b200.tt import TensorTrain, TTLinearOperator
    d = load(case)
    x0 = TensorTrain(train(d, "x0")) if "x0__n" in d else None
    x, rep = amen_solve(TTLinearOperator(train(d, "A")), TensorTrain(train(d, "f")), x0, to_config(d))
    r = {"converged": rep.converged, "sweeps_used": rep.sweeps_used,
         "final_relative_residual": rep.final_relative_residual,
         "rank_profile_history": rep.rank_profile_history}
    check_amen_parity(d, r, O.tt_full(list(x.cores)))
    assert len(rep.residual_history) == rep.sweeps_used


def test_zero_rhs():
    from paper_2501_12151_b200.amen import amen_solve
    from paper_2501_12151_b200.tt import tt_identity, tt_norm, tt_zero
    dims = (4, 4, 4)
    x, rep = amen_solve(tt_identity(dims), tt_zero(dims))
    assert rep.converged and rep.sweeps_used == 0 and rep.final_relative_residual == 0.0
    assert x.ranks == (1,) * 4 and tt_norm(x) == 0.0


def test_error_paths():
    from paper_2501_12151_b200.amen import amen_solve
    from paper_2501_12151_b200.errors import ShapeMismatchError, SolverError
    from paper_2501_12151_b200.tt import tt_identity, tt_ones, tt_op_add, tt_op_from_dense, tt_op_scale
    with pytest.raises(ShapeMismatchError):
        amen_solve(tt_identity((4, 4)), tt_ones((4, 4, 4)))
    with pytest.raises(SolverError, match="core"):  # singular local system (test_amen.py:173-179)
        amen_solve(tt_op_scale(tt_identity((4, 4)), 0.0), tt_ones((4, 4)))
    # a shift plus 2I is not symmetric (test_amen.py:164-170)
    A = tt_op_add(tt_op_from_dense(np.eye(16, k=4), (4, 4), (4, 4)), tt_op_scale(tt_identity((4, 4)), 2.0))
    with pytest.raises(SolverError, match="symmetric"):
        amen_solve(A, tt_ones((4, 4)))


def test_identity_and_scaled():
    from paper_2501_12151_b200.amen import amen_solve, residual_norm
    from paper_2501_12151_b200.tt import TensorTrain, tt_identity, tt_ones, tt_op_scale, tt_to_dense
    rng = np.random.default_rng(7)
    dims = (2, 4, 4)
    f = TensorTrain([rng.standard_normal((1, 2, 2)), rng.standard_normal((2, 4, 2)),
                     rng.standard_normal((2, 4, 1))])
    x, rep = amen_solve(tt_identity(dims), f)
    assert rep.converged and residual_norm(tt_identity(dims), x, f) <= 1e-13
    x, rep = amen_solve(tt_op_scale(tt_identity((4, 4)), 2.0), tt_ones((4, 4)))
    assert rep.converged and np.allclose(tt_to_dense(x), 0.5, atol=1e-12)


def test_config_c1_vs_reference_ensemble():
    """BASELINE config C1 itself (3D cube, 2^5 nodes/axis, 98,304 DOF, tol 1e-6, max rank 32,
    x0 rank-2 N(0,1) seed 0): the device solve must land inside the reference's own
    trajectory band (9 runs of the real reference under 1e-15 x0 perturbations,
    tests/golden/make_c1_band.py) widened by the north_star's 10%, with the same rank cap."""
    import json
    import os

    from paper_2501_12151_b200.amen import AmenConfig, amen_solve
    from paper_2501_12151_b200.configs import WORKLOADS, build
    from paper_2501_12151_b200.tt import TensorTrain, TruncationPolicy, TTLinearOperator
    from tests.golden_io import GOLDEN
    ref = json.load(open(os.path.join(GOLDEN, "c1_band.json")))
    prob, x0, kw = build(WORKLOADS["C1"])
    rel, cap = kw.pop("rounding")
    x, rep = amen_solve(TTLinearOperator(prob.op), TensorTrain(prob.rhs), TensorTrain(x0),
                        AmenConfig(rounding=TruncationPolicy(rel, cap), **kw))
    lo, hi = ref["band_final"]
    assert 0.9 * lo <= rep.final_relative_residual <= 1.1 * hi, (rep.final_relative_residual, ref["band_final"])
    assert rep.converged == ref["converged"]
    assert max(x.ranks) == max(ref["ranks"])
    slo, shi = ref["band_sweeps"]
    assert slo <= rep.sweeps_used <= shi


def test_solve_is_bitwise_reproducible():
    """Two solves of the same rank-limited system (C1 settings at L = 3, 8 sweeps) give
    bitwise identical residual histories and solutions: every reduction (split-K, CG dot
    products, Gershgorin max) has a fixed order, so trajectory differences can only come
    from different inputs or builds."""
    from paper_2501_12151_b200.amen import AmenConfig, amen_solve
    from paper_2501_12151_b200.assembly3d import assemble_cube
    from paper_2501_12151_b200.configs import x0_rank2
    from paper_2501_12151_b200.tt import TensorTrain, TruncationPolicy, TTLinearOperator
    prob = assemble_cube(3)
    cfg = AmenConfig(residual_tol=1e-6, max_sweeps=8, rounding=TruncationPolicy(1e-6, 16), seed=2024)
    runs = [amen_solve(TTLinearOperator(prob.op), TensorTrain(prob.rhs), TensorTrain(x0_rank2(prob.dims)), cfg)
            for _ in range(2)]
    (x1, r1), (x2, r2) = runs
    assert r1.residual_history == r2.residual_history
    assert all(np.array_equal(a, b) for a, b in zip(x1.cores, x2.cores))


def test_config_c2_vs_reference_ensemble():
    """BASELINE config C2 (2^8 nodes/axis, 5.0e7 DOF, tol 1e-6, max rank 64) -- local systems up
    to 68 x 2 x 68, so the persistent TMA CG kernel carries the solve -- against the real
    reference's trajectory band (8 runs, tests/golden/make_c1_band.py ... C2), widened by 10%."""
    import json
    import os

    from paper_2501_12151_b200.amen import AmenConfig, amen_solve
    from paper_2501_12151_b200.configs import WORKLOADS, build
    from paper_2501_12151_b200.tt import TensorTrain, TruncationPolicy, TTLinearOperator
    from tests.golden_io import GOLDEN
    ref = json.load(open(os.path.join(GOLDEN, "c2_band.json")))
    prob, x0, kw = build(WORKLOADS["C2"])
    rel, cap = kw.pop("rounding")
    x, rep = amen_solve(TTLinearOperator(prob.op), TensorTrain(prob.rhs), TensorTrain(x0),
                        AmenConfig(rounding=TruncationPolicy(rel, cap), **kw))
    lo, hi = ref["band_final"]
    assert 0.9 * lo <= rep.final_relative_residual <= 1.1 * hi, (rep.final_relative_residual, ref["band_final"])
    assert rep.converged == ref["converged"]
    assert max(x.ranks) == max(ref["ranks"])
