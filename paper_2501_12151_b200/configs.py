"""The BASELINE.json workloads as concrete problems (shared by bench.py and tests).

C1-C3: clamped unit cube, E=1, nu=0.3, body force (0,0,-1), 2^L nodes per axis
(the reference's node convention), tol 1e-6, max rank
32/64/96.  C5: two-layer E (1 / 10 split at z=0.5), traction (0,0,-1) on the
x=1 patch y,z in [0.25,0.75], tol 1e-7, max rank 192.  Solver settings follow
SURVEY.md section 8d: AmenConfig(residual_tol=tol,
rounding=TruncationPolicy(tol, max_rank), seed=2024), x0 = rank-2 N(0,1) TT from
default_rng(0) drawn core by core.  All data is synthetic (seeded) by construction.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .assembly3d import assemble_cube


@dataclass(frozen=True)
class Workload:
    name: str
    L: int
    tol: float
    max_rank: int
    load: str = "body"
    layers: tuple | None = None
    max_sweeps: int = 50

    @property
    def cells_per_axis(self) -> int:
        return 2 ** self.L - 1

    @property
    def dof(self) -> int:
        return 3 * 8 ** self.L


WORKLOADS = {
    "C1": Workload("C1", 5, 1e-6, 32),
    "C2": Workload("C2", 8, 1e-6, 64),
    "C3": Workload("C3", 10, 1e-6, 96),
    "C5": Workload("C5", 9, 1e-7, 192, load="patch", layers=(0.5, 1.0, 10.0)),
    # not a BASELINE config: the L <= 6 decompressed-field check of north_star (3 * 2^18 entries
    # fit tt_to_dense's cap), same cube problem as C1-C3
    "L6": Workload("L6", 6, 1e-6, 32),
}


def x0_rank2(dims, seed=0):
    """Rank-2 TT with N(0,1) cores from default_rng(seed), k = 0..K-1."""
    rng = np.random.default_rng(seed)
    K = len(dims)
    return [rng.standard_normal((1 if k == 0 else 2, dims[k], 1 if k == K - 1 else 2)) for k in range(K)]


def build(w: Workload, rounding: str = "device"):
    """Assemble (A cores, f cores, x0 cores, amen kwargs) for a workload (rounding: where the
    assembly's 1e-14 roundings run, assembly3d.assemble_cube)."""
    prob = assemble_cube(w.L, load=w.load, layers=w.layers, rounding=rounding)
    x0 = x0_rank2(prob.dims, 0)
    kw = dict(residual_tol=w.tol, max_sweeps=w.max_sweeps, rounding=(w.tol, w.max_rank), seed=2024)
    return prob, x0, kw


def c4_problem(r: int, d: int = 30, R: int = 16, seed: int = 1):
    """Config 4 (BASELINE.json): rng = default_rng(seed); MPO cores
    k = 0..d-1 of shape (1|R, 2, 2, R|1) first, then vector cores (1|r, 2, r|1), all
    standard_normal * r**-0.5 (the literal reading of N(0, 1/r), MPO cores included)."""
    rng = np.random.default_rng(seed)
    s = r ** -0.5
    op = [rng.standard_normal((1 if k == 0 else R, 2, 2, 1 if k == d - 1 else R)) * s for k in range(d)]
    x = [rng.standard_normal((1 if k == 0 else r, 2, 1 if k == d - 1 else r)) * s for k in range(d)]
    return op, x
