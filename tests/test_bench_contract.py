"""CPU checks of bench.py's bookkeeping (VERDICT r1 'Bench bookkeeping')."""
import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _bench():
    sys.argv = ["bench.py"]
    import bench
    return bench


def test_recorded_trajectory_belongs_to_this_engine_build():
    """--impl reference extrapolates over profiles/trajectory_C3.json; it must have been
    recorded by the engine built from the current sources, and describe ONE solve."""
    b = _bench()
    t = json.load(open(os.path.join(ROOT, "profiles", "trajectory_C3.json")))
    assert t["source_sha256"] == b.source_digest(), "re-record profiles/trajectory_C3.json with bench.py"
    tr = np.array(t["trace"])
    assert int(tr[:, 10].sum()) == t["cg_iterations"]
    assert tr[:, 0].max() == t["sweeps"] and tr[:, 0].min() == 1  # one solve's sweeps 1..S
    K = len(t["x_ranks"]) - 1
    assert len(tr) <= t["sweeps"] * K


def test_both_arms_share_the_config():
    b = _bench()
    from paper_2501_12151_b200.configs import WORKLOADS
    w = WORKLOADS["C3"]
    cfg = b.workload_config(w)
    assert "assembly_s" not in cfg and "parallelism" not in cfg
    assert cfg["workload"].startswith("C3:")
