"""Run the same AMEn solve several times in one process and compare the residual
histories bit for bit: python tools/determinism.py [C1|C2|C3] [max_sweeps] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2501_12151_b200.amen import AmenConfig, amen_solve  # noqa: E402
from paper_2501_12151_b200.configs import WORKLOADS, build  # noqa: E402
from paper_2501_12151_b200.tt import TensorTrain, TruncationPolicy, TTLinearOperator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
prob, x0, kw = build(WORKLOADS[name])
kw["max_sweeps"] = sweeps
rel, cap = kw.pop("rounding")
cfg = AmenConfig(rounding=TruncationPolicy(rel, cap), **kw)
hist = []
from paper_2501_12151_b200 import _native as nat  # noqa: E402
perturb = os.environ.get("PERTURB_POOL") == "1"
for r in range(reps):
    if perturb and r > 0:  # change the memory pool's layout between runs (stale contents differ)
        ctx = nat.default_context()
        ctx.flush_l2()
        import torch
        junk = torch.full((int(3e7),), float("nan"), dtype=torch.float64, device="cuda")
        del junk
    if os.environ.get("PROFILE_SECOND") == "1" and r > 0:
        nat.default_context().set_profiling(True)
    x, rep = amen_solve(TTLinearOperator(prob.op), TensorTrain(prob.rhs), TensorTrain(x0), cfg)
    hist.append(np.array(rep.residual_history))
    print(r, rep.sweeps_used, repr(rep.final_relative_residual), flush=True)
same = all(len(h) == len(hist[0]) and np.array_equal(h, hist[0]) for h in hist)
print("bitwise identical residual histories:", same)
if not same:
    for h in hist:
        print([f"{v:.17g}" for v in h[:12]])
