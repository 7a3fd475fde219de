"""Decompressed-field parity at L <= 6 (north_star criterion 4).

C1 (L = 5, 98,304 entries) and the L = 6 cube (786,432 entries; configs.WORKLOADS["L6"]) are
rank-limited (max rank 32): neither the device nor the reference converges to tol = 1e-6 (final
residuals ~0.05 / ~0.17), so "field within 10 x tol" cannot hold even between two runs of the
reference: nine reference runs (x0 perturbed by 1e-15; tests/golden/make_field_band.py) spread
1.6e-5 .. 2.0e-5 (C1) and 2.0e-5 .. 3.6e-5 (L6) in relative L2 around each other.  The device
field is held to that ensemble: its distance to reference member 0 must not exceed 1.25x the
ensemble's largest pairwise distance."""
import json
import os

import numpy as np
import pytest

from tests.golden_io import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["C1", "L6"])
def test_field_vs_reference_ensemble(name):
    from paper_2501_12151_b200.amen import AmenConfig, amen_solve
    from paper_2501_12151_b200.configs import WORKLOADS, build
    from paper_2501_12151_b200.tt import TensorTrain, TruncationPolicy, TTLinearOperator, tt_to_dense
    band = json.load(open(os.path.join(GOLDEN, f"field_{name}.json")))
    z = np.load(os.path.join(GOLDEN, f"field_{name}.npz"))
    ref = tt_to_dense(TensorTrain([z[f"arr_{k}"] for k in range(len(z.files))]))
    prob, x0, kw = build(WORKLOADS[name])
    rel, cap = kw.pop("rounding")
    x, rep = amen_solve(TTLinearOperator(prob.op), TensorTrain(prob.rhs), TensorTrain(x0),
                        AmenConfig(rounding=TruncationPolicy(rel, cap), **kw))
    u = tt_to_dense(x)
    assert u.size == band["entries"]
    d = float(np.linalg.norm(u - ref) / np.linalg.norm(ref))
    print(f"{name}: device field vs reference member 0: {d:.3e} (ensemble pairwise max "
          f"{band['pairwise_max']:.3e}, median {band['pairwise_median']:.3e}; 10 x tol = {10 * band['tol']:.0e})")
    assert d <= 1.25 * band["pairwise_max"], d
    # and the solve itself sits inside the ensemble's residual band (+-10%)
    lo, hi = min(band["finals"]), max(band["finals"])
    assert 0.9 * lo <= rep.final_relative_residual <= 1.1 * hi
