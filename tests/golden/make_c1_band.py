"""Reference ensemble for configs C1 / C2.  Config C1 (BASELINE configs[0]: 3D cube, 2^5 nodes per axis, tol 1e-6,
max rank 32, x0 rank-2 N(0,1) seed 0, AmenConfig seed 2024), run with the REAL reference in the
build container (the reference is pure Python; ~20 min per run on one core):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c1_band.py MEMBER [C1|C2]  # 0..8
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c1_band.py combine [C1|C2]

Member 0 is the unperturbed solve; members 1..8 perturb x0 by 1e-15 relative (the same
trajectory-sensitivity ensemble as make_golden.py's amen fixtures).  `combine` writes the
small summary tests/golden/c1_band.json that tests/test_gpu_amen.py checks the device C1
solve against."""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import ttfem.tt as rtt  # noqa: E402
import ttfem.amen as ram  # noqa: E402

rtt._ALLOWED_MODES = (2, 3, 4, 8, 9)

from paper_2501_12151_b200.configs import WORKLOADS, build  # noqa: E402


def member(i, cfg_name="C1"):
    prob, x0, kw = build(WORKLOADS[cfg_name], rounding="host")
    rel, cap = kw.pop("rounding")
    cfg = ram.AmenConfig(rounding=rtt.TruncationPolicy(rel, cap), **kw)
    if i > 0:
        prng = np.random.default_rng(1000 + i - 1)
        x0 = [c * (1 + 1e-15 * prng.standard_normal(c.shape)) for c in x0]
    t0 = time.time()
    x, rep = ram.amen_solve(rtt.TTLinearOperator(prob.op), rtt.TensorTrain(prob.rhs), x0=rtt.TensorTrain(x0),
                            config=cfg)
    out = {"member": i, "seconds": time.time() - t0, "converged": bool(rep.converged),
           "sweeps": int(rep.sweeps_used), "final": float(rep.final_relative_residual),
           "res_hist": [float(v) for v in rep.residual_history], "ranks": list(map(int, x.ranks))}
    json.dump(out, open(os.path.join("/tmp", f"{cfg_name.lower()}_member_{i}.json"), "w"))
    print(out)


def combine(cfg_name="C1"):
    tag = cfg_name.lower()
    ms = [json.load(open(os.path.join("/tmp", f"{tag}_member_{i}.json"))) for i in range(9)
          if os.path.exists(os.path.join("/tmp", f"{tag}_member_{i}.json"))]
    m0 = [m for m in ms if m["member"] == 0][0]
    d = {"config": cfg_name, "members": len(ms), "reference_seconds_per_solve": float(np.mean([m["seconds"] for m in ms])),
         "final": m0["final"], "sweeps": m0["sweeps"], "converged": m0["converged"], "ranks": m0["ranks"],
         "res_hist": m0["res_hist"],
         "band_final": [min(m["final"] for m in ms), max(m["final"] for m in ms)],
         "band_sweeps": [min(m["sweeps"] for m in ms), max(m["sweeps"] for m in ms)]}
    json.dump(d, open(os.path.join(HERE, f"{tag}_band.json"), "w"), indent=1)
    print(d["band_final"], d["band_sweeps"])


if __name__ == "__main__":
    name = sys.argv[2] if len(sys.argv) > 2 else "C1"
    combine(name) if sys.argv[1] == "combine" else member(int(sys.argv[1]), name)
