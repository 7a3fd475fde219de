"""Reference field ensembles for the L <= 6 field check (north_star criterion 4).

For C1 (L = 5, max rank 32) and the L = 6 cube (max rank 32) -- both rank-limited, so neither
converges to tol and the "field within 10 x tol" criterion cannot be met by the reference itself
-- run 9 members of the UNMODIFIED reference amen_solve (member 0 unperturbed, members 1..8 with
x0 perturbed by 1e-15 relative) and record, for every member, its decompressed field
(ttfem.tt.tt_to_dense), its distance to member 0, and the ensemble's pairwise spread.  The GPU
test compares the device field with member 0's by the same measure.

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_field_band.py MEMBER C1|L6
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_field_band.py combine C1|L6

Writes tests/golden/field_<cfg>.npz (member 0's solution cores) and field_<cfg>.json (spread).
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

rtt._ALLOWED_MODES = (2, 3, 4, 8, 9)

from paper_2501_12151_b200.configs import WORKLOADS, build  # noqa: E402

OUT = os.environ.get("BAND_TMP", "/tmp/band")


def member(i, name):
    prob, x0, kw = build(WORKLOADS[name], rounding="host")
    rel, cap = kw.pop("rounding")
    cfg = ram.AmenConfig(rounding=rtt.TruncationPolicy(rel, cap), **kw)
    if i > 0:
        prng = np.random.default_rng(1000 + i - 1)
        x0 = [c * (1 + 1e-15 * prng.standard_normal(c.shape)) for c in x0]
    t0 = time.time()
    x, rep = ram.amen_solve(rtt.TTLinearOperator(prob.op), rtt.TensorTrain(prob.rhs), x0=rtt.TensorTrain(x0),
                            config=cfg)
    os.makedirs(OUT, exist_ok=True)
    np.savez(os.path.join(OUT, f"field_{name}_{i}.npz"), *x.cores)
    out = {"member": i, "seconds": time.time() - t0, "converged": bool(rep.converged), "sweeps": rep.sweeps_used,
           "final": float(rep.final_relative_residual)}
    json.dump(out, open(os.path.join(OUT, f"field_{name}_{i}.json"), "w"))
    print(out, flush=True)


def combine(name):
    cores, meta, fields = [], [], []
    for i in range(9):
        p = os.path.join(OUT, f"field_{name}_{i}.npz")
        if not os.path.exists(p):
            continue
        z = np.load(p)
        c = [z[f"arr_{k}"] for k in range(len(z.files))]
        cores.append(c)
        meta.append(json.load(open(os.path.join(OUT, f"field_{name}_{i}.json"))))
        fields.append(rtt.tt_to_dense(rtt.TensorTrain(c)))
    u0 = fields[0]
    d0 = [float(np.linalg.norm(u - u0) / np.linalg.norm(u0)) for u in fields[1:]]
    pair = [float(np.linalg.norm(a - b) / np.linalg.norm(b)) for j, a in enumerate(fields) for b in fields[j + 1:]]
    np.savez(os.path.join(HERE, f"field_{name}.npz"), *cores[0])
    d = {"config": name, "members": len(fields), "tol": WORKLOADS[name].tol,
         "finals": [m["final"] for m in meta], "sweeps": [m["sweeps"] for m in meta],
         "converged": [m["converged"] for m in meta],
         "dist_to_member0": d0, "pairwise_max": max(pair), "pairwise_median": float(np.median(pair)),
         "field_norm": float(np.linalg.norm(u0)), "entries": int(u0.size)}
    json.dump(d, open(os.path.join(HERE, f"field_{name}.json"), "w"), indent=1)
    print(d)


if __name__ == "__main__":
    combine(sys.argv[2]) if sys.argv[1] == "combine" else member(int(sys.argv[1]), sys.argv[2])
