"""Readers for the frozen reference fixtures in tests/golden (see make_golden.py)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def train(d, name):
    n = int(d[f"{name}__n"])
    return [d[f"{name}__{k}"] for k in range(n)]


def amen_config(d):
    rel, cap = d["cfg_rounding"]
    return {
        "residual_tol": float(d["cfg_residual_tol"]),
        "max_sweeps": int(d["cfg_max_sweeps"]),
        "enrichment_rank": int(d["cfg_enrichment_rank"]),
        "local_solver": str(d["cfg_local_solver"]),
        "direct_dim_cap": int(d["cfg_direct_dim_cap"]),
        "local_iter_cap": int(d["cfg_local_iter_cap"]),
        "rounding": (float(rel), None if cap < 0 else int(cap)),
        "seed": int(d["cfg_seed"]),
        "stagnation_strikes": int(d["cfg_stagnation_strikes"]),
    }


AMEN_CASES = sorted(f for f in os.listdir(GOLDEN) if f.startswith("amen_") and f.endswith(".npz"))
