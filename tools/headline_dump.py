"""GPU side of the headline parity pins (tests/test_gpu_headline.py).

    python tools/headline_dump.py inputs C3|C5    # device-assembled A, f -> gpurun_out/<cfg>_{op,rhs}.qtt1
    python tools/headline_dump.py full C3|C5      # full solve, x saved as gpurun_out/<cfg>_x.qtt1
    python tools/headline_dump.py bounded C3|C5 K # K sweeps, stagnation_strikes=0 (the ensemble pin)
    QTT_DUMP_STEP=sweep,core,path python tools/headline_dump.py full C3   # + core-step state dump

Prints one JSON line per run (final residual, sweeps, rank history, per-sweep estimates)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2501_12151_b200 import _native as nat  # noqa: E402
from paper_2501_12151_b200.amen import AmenConfig, amen_solve  # noqa: E402
from paper_2501_12151_b200.configs import WORKLOADS, build  # noqa: E402
from paper_2501_12151_b200.serialize import save_tt  # noqa: E402
from paper_2501_12151_b200.tt import TensorTrain, TruncationPolicy, TTLinearOperator  # noqa: E402


def main():
    mode, name = sys.argv[1], sys.argv[2]
    prob, x0, kw = build(WORKLOADS[name])
    if mode == "inputs":  # the device-assembled operator and load, for the reference-side scripts
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        save_tt(TTLinearOperator(prob.op), os.path.join(ROOT, "gpurun_out", f"{name.lower()}_op.qtt1"))
        save_tt(TensorTrain(prob.rhs), os.path.join(ROOT, "gpurun_out", f"{name.lower()}_rhs.qtt1"))
        print(json.dumps({"mode": mode, "config": name, "op_ranks": list(prob.op_ranks)}))
        return
    rel, cap = kw.pop("rounding")
    if mode == "bounded":
        kw.update(max_sweeps=int(sys.argv[3]), stagnation_strikes=0)
    cfg = AmenConfig(rounding=TruncationPolicy(rel, cap), **kw)
    ctx = nat.default_context()
    t0 = time.perf_counter()
    x, rep = amen_solve(TTLinearOperator(prob.op), TensorTrain(prob.rhs), TensorTrain(x0), cfg, ctx=ctx)
    dt = time.perf_counter() - t0
    out = {"mode": mode, "config": name, "max_sweeps": cfg.max_sweeps, "seconds": dt,
           "converged": rep.converged, "sweeps": rep.sweeps_used, "final": rep.final_relative_residual,
           "res_hist": list(rep.residual_history), "rank_hist": [list(r) for r in rep.rank_profile_history]}
    if mode == "full":
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        save_tt(x, os.path.join(ROOT, "gpurun_out", f"{name.lower()}_x.qtt1"))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
