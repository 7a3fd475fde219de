"""Bounded-sweep reference ensembles for the headline configs C3 and C5.

The full C3/C5 solves (45-50 sweeps at ranks ~100/196) are out of reach for the pure-Python
reference (SURVEY.md 8d estimates ~6 h / ~1.5 days per solve), and the sweep is chaotic in
floating point, so the pin is an ensemble of the UNMODIFIED reference
(`ttfem.amen.amen_solve`, /root/reference/pkg/src/ttfem/amen.py:394-510) stopped after K sweeps with
`stagnation_strikes=0` (no plateau certifications, no z re-draws: a fixed amount of work on both
sides).  Member 0 is the unperturbed problem (x0 = rank-2 N(0,1) from default_rng(0)); members
1..8 perturb x0 by 1e-15 relative.  Run in the build container (the reference is importable
there, not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_bounded_band.py MEMBER C3|C5 K      # MEMBER = 0..8
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bounded_band.py combine C3|C5 K

`combine` writes tests/golden/<cfg>_k<K>_band.json (residual band, per-sweep estimate bands,
rank profiles of every member), checked by tests/test_gpu_headline.py.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import ttfem.amen as ram  # noqa: E402
import ttfem.tt as rtt  # noqa: E402

rtt._ALLOWED_MODES = (2, 3, 4, 8, 9)  # the 3-component leading core

from paper_2501_12151_b200.configs import WORKLOADS, build, x0_rank2  # noqa: E402
from tests.golden_io import headline_inputs  # noqa: E402

OUT = os.environ.get("BAND_TMP", "/tmp/band2")


def member(i, cfg_name, k):
    # the B200's own (device-assembled, deterministic) operator and load, committed as QTT1
    op, rhs = headline_inputs(cfg_name)
    w = WORKLOADS[cfg_name]
    x0 = x0_rank2([c.shape[1] for c in rhs], 0)
    kw = dict(residual_tol=w.tol, max_sweeps=w.max_sweeps, rounding=(w.tol, w.max_rank), seed=2024)
    rel, cap = kw.pop("rounding")
    kw.update(max_sweeps=k, stagnation_strikes=0)
    cfg = ram.AmenConfig(rounding=rtt.TruncationPolicy(rel, cap), **kw)
    if i > 0:
        prng = np.random.default_rng(1000 + i - 1)
        x0 = [c * (1 + 1e-15 * prng.standard_normal(c.shape)) for c in x0]
    t0 = time.time()
    x, rep = ram.amen_solve(rtt.TTLinearOperator(op), rtt.TensorTrain(rhs), x0=rtt.TensorTrain(x0),
                            config=cfg)
    out = {"member": i, "seconds": time.time() - t0, "converged": bool(rep.converged),
           "sweeps": int(rep.sweeps_used), "final": float(rep.final_relative_residual),
           "res_hist": [float(v) for v in rep.residual_history],
           "rank_hist": [list(map(int, r)) for r in rep.rank_profile_history]}
    os.makedirs(OUT, exist_ok=True)
    json.dump(out, open(os.path.join(OUT, f"{cfg_name.lower()}_k{k}_member_{i}.json"), "w"))
    print(json.dumps({kk: out[kk] for kk in ("member", "seconds", "sweeps", "final")}))


def combine(cfg_name, k):
    tag = f"{cfg_name.lower()}_k{k}"
    ms = [json.load(open(os.path.join(OUT, f"{tag}_member_{i}.json"))) for i in range(9)
          if os.path.exists(os.path.join(OUT, f"{tag}_member_{i}.json"))]
    m0 = [m for m in ms if m["member"] == 0][0]
    est = np.array([m["res_hist"] for m in ms])
    d = {"config": cfg_name, "max_sweeps": k, "stagnation_strikes": 0, "members": len(ms),
         "reference_seconds_per_solve": float(np.mean([m["seconds"] for m in ms])),
         "final": m0["final"], "res_hist": m0["res_hist"], "rank_hist": m0["rank_hist"],
         "band_final": [min(m["final"] for m in ms), max(m["final"] for m in ms)],
         "band_est": [est.min(axis=0).tolist(), est.max(axis=0).tolist()],
         "member_finals": [m["final"] for m in ms],
         "member_final_ranks": [m["rank_hist"][-1] for m in ms],
         "member_rank_hist": [m["rank_hist"] for m in ms]}
    json.dump(d, open(os.path.join(HERE, f"{tag}_band.json"), "w"))
    print(d["band_final"], "ranks equal across members:",
          all(r == ms[0]["rank_hist"] for r in (m["rank_hist"] for m in ms)))


if __name__ == "__main__":
    cfg_name = sys.argv[2]
    k = int(sys.argv[3])
    combine(cfg_name, k) if sys.argv[1] == "combine" else member(int(sys.argv[1]), cfg_name, k)
