"""Config 4 (kernel microbench on random TT data): the matvec sweep
(right-env pre-pass + local matvec + left env per core) and tt_round(tt_apply(A, x)).

CPU: the oracle against the reference's own outputs (tests/golden/c4_small.npz).
GPU: the device sweep / apply / round against the fixture and the oracle, at the
fixture sizes and at the config's own shapes (d = 30, R = 16, r = 32).  Bar: <= 1e-12
relative for the contractions (FP64), equal ranks and <= 1e-12 relative for rounding."""
import numpy as np
import pytest

from oracle import qtt_oracle as O
from tests.golden_io import load, train

TOL = 1e-12


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def test_c4_generator_shapes():
    from paper_2501_12151_b200.configs import c4_problem
    op, x = c4_problem(32)
    assert len(op) == len(x) == 30
    assert op[0].shape == (1, 2, 2, 16) and op[5].shape == (16, 2, 2, 16) and op[-1].shape == (16, 2, 2, 1)
    assert x[0].shape == (1, 2, 32) and x[7].shape == (32, 2, 32) and x[-1].shape == (32, 2, 1)
    # same draws as the fixture's generator call
    d = load("c4_small.npz")
    op_a, x_a = c4_problem(6, d=10, R=4, seed=1)
    for c, r in zip(op_a + x_a, train(d, "a_A") + train(d, "a_x")):
        assert np.array_equal(c, r)


@pytest.mark.parametrize("tag", ["a", "b"])
def test_oracle_sweep_and_round_vs_reference(tag):
    d = load("c4_small.npz")
    A, x = train(d, f"{tag}_A"), train(d, f"{tag}_x")
    for y, r in zip(O.matvec_sweep(A, x), train(d, f"{tag}_y")):
        assert y.shape == r.shape and rel(y, r) <= 1e-13
    ap = O.tt_apply(A, x)
    if f"{tag}_apply__n" in d:
        for c, r in zip(ap, train(d, f"{tag}_apply")):
            assert c.shape == r.shape and rel(c, r) <= 1e-15
    rd = O.tt_round(ap, 1e-8)
    ref = train(d, f"{tag}_round")
    assert [c.shape for c in rd] == [c.shape for c in ref]
    assert rel(O.tt_full(rd), O.tt_full(ref)) <= 1e-12


@pytest.fixture(scope="module")
def K():
    from paper_2501_12151_b200 import kernels
    return kernels


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["a", "b"])
def test_gpu_sweep_apply_round_vs_reference(K, tag):
    from paper_2501_12151_b200 import tt
    d = load("c4_small.npz")
    A, x = train(d, f"{tag}_A"), train(d, f"{tag}_x")
    ys, times = K.matvec_sweep(tt.TTLinearOperator(A), tt.TensorTrain(x), timing=True, split_timing=True)
    for y, r in zip(ys, train(d, f"{tag}_y")):
        assert y.shape == r.shape and rel(y, r) <= TOL
    assert times["sweep_ms"] > 0 and times["k1_flops"] > 0
    Aop, X = tt.TTLinearOperator(A), tt.TensorTrain(x)
    ap = tt.tt_apply(Aop, X, None)
    for c, r in zip(ap.cores, O.tt_apply(A, x)):
        assert c.shape == r.shape and rel(c, r) <= 1e-15
    rd = tt.tt_apply(Aop, X, tt.TruncationPolicy(1e-8))
    ref = train(d, f"{tag}_round")
    assert [c.shape for c in rd.cores] == [c.shape for c in ref]
    assert rel(O.tt_full(rd.cores), O.tt_full(ref)) <= 1e-12


@pytest.mark.gpu
def test_gpu_sweep_config4_shapes_r32(K):
    """d = 30, R = 16, r = 32 (the config's smallest rank): every y_k vs the oracle."""
    from paper_2501_12151_b200 import tt
    from paper_2501_12151_b200.configs import c4_problem
    op, x = c4_problem(32)
    ys, _ = K.matvec_sweep(tt.TTLinearOperator(op), tt.TensorTrain(x))
    for k, (y, r) in enumerate(zip(ys, O.matvec_sweep(op, x))):
        assert y.shape == r.shape and rel(y, r) <= TOL, k


@pytest.mark.gpu
def test_gpu_sweep_rejects_bad_shapes(K):
    from paper_2501_12151_b200 import tt
    from paper_2501_12151_b200.errors import ShapeMismatchError
    from paper_2501_12151_b200.configs import c4_problem
    op, x = c4_problem(4, d=5, R=3)
    with pytest.raises(ShapeMismatchError):
        K.matvec_sweep(tt.TTLinearOperator(op[:4]), tt.TensorTrain(x))


@pytest.mark.gpu
def test_gpu_round_config4_r32_vs_oracle():
    """tt_round(tt_apply(A, x, None), 1e-8) at the config's r = 32 (bond 512, multi-CTA QR and
    block-Jacobi SVD): ranks equal to the oracle's, difference <= 1e-12 relative (TT norm)."""
    from paper_2501_12151_b200 import tt
    from paper_2501_12151_b200.configs import c4_problem
    op, x = c4_problem(32)
    y = tt.tt_apply(tt.TTLinearOperator(op), tt.TensorTrain(x), tt.TruncationPolicy(1e-8))
    ref = O.tt_round(O.tt_apply(op, x), 1e-8)
    assert [c.shape for c in y.cores] == [c.shape for c in ref]
    diff = O.tt_norm(O.tt_sub(list(y.cores), ref))
    assert diff <= 1e-12 * O.tt_norm(ref)


@pytest.mark.gpu
def test_gpu_round_large_bond_truncating_vs_oracle():
    """A rank-deficient large bond (x + x at bond 600 = 2 x 300): the certified no-truncation
    path must refuse and the SVD path truncate to the oracle's ranks."""
    from paper_2501_12151_b200 import tt
    rng = np.random.default_rng(7)
    dims = (2, 2, 2, 2, 2, 2, 2, 2, 2, 2)
    ranks = [1, 2, 4, 8, 16, 300, 16, 8, 4, 2, 1]
    x = [rng.standard_normal((ranks[k], 2, ranks[k + 1])) / np.sqrt(ranks[k]) for k in range(len(dims))]
    xx = O.tt_add(x, x)
    y = tt.tt_round(tt.TensorTrain(xx), tt.TruncationPolicy(1e-10))
    ref = O.tt_round(xx, 1e-10)
    assert [c.shape for c in y.cores] == [c.shape for c in ref]
    assert O.tt_norm(O.tt_sub(list(y.cores), ref)) <= 1e-12 * O.tt_norm(ref)


@pytest.mark.gpu
def test_gpu_sweep_tma_gemm_sizes():
    """Ranks large enough for the TMA GEMM path (local-matvec step 1 with a transposed v, step 3
    and the left-environment update): every y_k of the sweep vs the oracle at <= 1e-12."""
    from paper_2501_12151_b200 import kernels, tt
    from paper_2501_12151_b200.configs import c4_problem
    op, x = c4_problem(128, d=9)
    ys, _ = kernels.matvec_sweep(tt.TTLinearOperator(op), tt.TensorTrain(x))
    for k, (y, r) in enumerate(zip(ys, O.matvec_sweep(op, x))):
        assert y.shape == r.shape and rel(y, r) <= TOL, k
