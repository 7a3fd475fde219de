import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2501_12151_b200 import _native as nat
from paper_2501_12151_b200.amen import AmenConfig, amen_solve_device, random_draws
from paper_2501_12151_b200.configs import WORKLOADS, build
from paper_2501_12151_b200.tt import DeviceTrain, TensorTrain, TruncationPolicy, TTLinearOperator
name = sys.argv[1]; sweeps = int(sys.argv[2])
prob, x0, kw = build(WORKLOADS[name]); kw["max_sweeps"] = sweeps
rel, cap = kw.pop("rounding"); cfg = AmenConfig(rounding=TruncationPolicy(rel, cap), **kw)
A, f, X0 = TTLinearOperator(prob.op), TensorTrain(prob.rhs), TensorTrain(x0)
ctx = nat.default_context()
draws = random_draws(A, f.dims, cfg)
dA, df, dx0 = (DeviceTrain.upload(t.cores, ctx) for t in (A, f, X0))
a0 = [c.copy() for c in dA.cores()]; f0 = [c.copy() for c in df.cores()]; x00 = [c.copy() for c in dx0.cores()]
for r in range(3):
    dx, info = amen_solve_device(dA, df, dx0, cfg, draws, A.order, ctx)
    print(r, info["sweeps_used"], repr(info["final_relative_residual"]), flush=True)
    print("  A unchanged:", all(np.array_equal(a, b) for a, b in zip(a0, dA.cores())),
          "f unchanged:", all(np.array_equal(a, b) for a, b in zip(f0, df.cores())),
          "x0 unchanged:", all(np.array_equal(a, b) for a, b in zip(x00, dx0.cores())), flush=True)
