"""Run one BASELINE workload on the GPU (and optionally the CPU oracle) and print a
JSON summary: python tools/run_config.py C1 [--oracle] [--profile]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2501_12151_b200 import _native as nat  # noqa: E402
from paper_2501_12151_b200.amen import AmenConfig, amen_solve  # noqa: E402
from paper_2501_12151_b200.configs import WORKLOADS, build  # noqa: E402
from paper_2501_12151_b200.tt import TensorTrain, TruncationPolicy, TTLinearOperator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--max-sweeps", type=int, default=None)
    a = ap.parse_args()
    w = WORKLOADS[a.name]
    t0 = time.perf_counter()
    prob, x0, kw = build(w)
    t_asm = time.perf_counter() - t0
    if a.max_sweeps:
        kw["max_sweeps"] = a.max_sweeps
    rel, cap = kw.pop("rounding")
    cfg = AmenConfig(rounding=TruncationPolicy(rel, cap), **kw)
    A, f, X0 = TTLinearOperator(prob.op), TensorTrain(prob.rhs), TensorTrain(x0)
    ctx = nat.default_context()
    ctx.set_profiling(a.profile, phases=a.profile)
    # warm-up on a tiny problem (module load, kernel attributes)
    ctx.reset_stats()
    t0 = time.perf_counter()
    x, rep = amen_solve(A, f, X0, cfg, ctx=ctx)
    t_gpu = time.perf_counter() - t0
    st = ctx.stats()
    out = {"workload": a.name, "L": w.L, "dof": w.dof, "op_ranks_max": max(prob.op_ranks),
           "assembly_s": t_asm, "gpu_s": t_gpu, "converged": rep.converged, "sweeps": rep.sweeps_used,
           "final": rep.final_relative_residual, "max_rank": max(x.ranks),
           "res_hist": [float(f"{v:.3e}") for v in rep.residual_history], "stats": st}
    if st["k1_ms"] > 0:
        out["k1_tflops"] = st["k1_timed_flops"] / st["k1_ms"] / 1e9
    if st["env_ms"] > 0:
        out["env_tflops"] = st["env_timed_flops"] / st["env_ms"] / 1e9
    if a.oracle:
        from oracle import qtt_oracle as O
        ocfg = dict(kw)
        ocfg["rounding"] = (rel, cap)
        t0 = time.perf_counter()
        xo, ro = O.amen_solve(prob.op, prob.rhs, x0, ocfg)
        out["oracle_s"] = time.perf_counter() - t0
        out["oracle_final"] = ro["final_relative_residual"]
        out["oracle_sweeps"] = ro["sweeps_used"]
        out["oracle_converged"] = ro["converged"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
