"""Config-4 kernel microbench (BASELINE.json configs[3]) on the GPU.

    python tools/c4_bench.py [--ranks 32,64,128,256] [--reps 3] [--out FILE]

For each rank r: A = MPO (d=30, 2x2 modes, rank 16), x = TT (d=30, mode 2, rank r),
all cores N(0, 1/r) from default_rng(1) (configs.c4_problem), device-resident.
Measured (CUDA events, median of --reps after one warm-up):
  (i)  the right-environment pre-pass, then one L->R sweep of local matvecs (K1) plus
       left environment updates (K2), with K1/K2 TFLOP/s from per-launch-group events
       against the measured FP64 DMMA peak;
  (ii) tt_apply(A, x, None) (Kronecker cores; HBM-bound: bytes = output written + inputs
       read) and tt_round(., 1e-8) where the device SVD supports the bond size.
Prints one JSON line per rank (and writes them to --out)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2501_12151_b200 import _native as nat  # noqa: E402
from paper_2501_12151_b200 import kernels  # noqa: E402
from paper_2501_12151_b200.configs import c4_problem  # noqa: E402
from paper_2501_12151_b200.tt import DeviceTrain  # noqa: E402


def peaks():
    fp64 = None
    p = os.path.join(ROOT, "profiles", "fp64_peaks_r01.jsonl")
    if os.path.exists(p):
        for line in open(p):
            d = json.loads(line)
            if d.get("what") == "dmma_m8n8k4":
                fp64 = max(fp64 or 0.0, d["tflops"])
    hbm = None
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        hbm = json.load(open(mp)).get("hbm_gbs")
    return fp64 or 37.1, hbm or 6516.7


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", default="32,64,128,256")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--round-max-bond", type=int, default=1024,
                    help="skip tt_round when R*r exceeds this (device SVD limit)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    fp64_peak, hbm_peak = peaks()
    ctx = nat.default_context()
    lines = []
    for r in [int(v) for v in a.ranks.split(",")]:
        op, x = c4_problem(r)
        dA, dx = DeviceTrain.upload(op, ctx), DeviceTrain.upload(x, ctx)
        kernels.matvec_sweep(dA, dx, ctx=ctx, timing=True, return_y=False)  # warm-up
        runs, split = [], []
        for _ in range(a.reps):
            ctx.flush_l2()
            runs.append(kernels.matvec_sweep(dA, dx, ctx=ctx, timing=True, return_y=False)[1])
        for _ in range(a.reps):
            split.append(kernels.matvec_sweep(dA, dx, ctx=ctx, timing=True, split_timing=True,
                                              return_y=False)[1])
        med = lambda rs, k: float(np.median([t[k] for t in rs]))  # noqa: E731
        t = runs[0]
        k1f, k2f, prf = t["k1_flops"], t["k2_flops"], t["prepass_flops"]
        sweep_ms, pre_ms = med(runs, "sweep_ms"), med(runs, "prepass_ms")
        k1_ms, k2_ms = med(split, "k1_ms"), med(split, "k2_ms")
        out = {"config": "C4", "r": r, "d": 30, "R": 16,
               "sweep": {"ms": sweep_ms, "tflops": (k1f + k2f) / sweep_ms / 1e9,
                         "k1_gflop": k1f / 1e9, "k2_gflop": k2f / 1e9,
                         "k1_ms": k1_ms, "k1_tflops": k1f / k1_ms / 1e9,
                         "k1_frac_fp64_peak": k1f / k1_ms / 1e9 / fp64_peak,
                         "k2_ms": k2_ms, "k2_tflops": k2f / k2_ms / 1e9},
               "prepass": {"ms": pre_ms, "tflops": prf / pre_ms / 1e9},
               "fp64_peak_tflops": fp64_peak}
        # (ii) TT-matvec then rounding
        import ctypes
        h = ctypes.c_void_p()
        nat.call("qtt_tt_apply", ctx.handle, dA.handle, dx.handle, ctypes.byref(h))  # warm-up
        y = DeviceTrain(h, ctx)  # the product's cores, allocated once outside the timed region
        import torch
        stream = torch.cuda.ExternalStream(ctx.stream)
        ts = []
        for _ in range(a.reps):
            ctx.flush_l2()
            ctx.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            nat.call("qtt_tt_apply_into", ctx.handle, dA.handle, dx.handle, y.handle)
            e1.record(stream)
            ctx.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        ta = float(np.min(ts))
        out_bytes = sum((o.shape[0] * v.shape[0]) * 2 * (o.shape[3] * v.shape[2]) * 8 for o, v in zip(op, x))
        in_bytes = sum(o.size * 8 + v.size * 8 for o, v in zip(op, x))
        out["apply"] = {"ms": ta * 1e3, "bytes": out_bytes + in_bytes,
                        "gbs": (out_bytes + in_bytes) / ta / 1e9, "frac_hbm_peak": (out_bytes + in_bytes) / ta / 1e9 / hbm_peak,
                        "timing": "CUDA events on the engine stream around qtt_tt_apply_into (one launch for all 30 cores, output preallocated), L2 flushed, min of reps"}
        if 16 * r <= a.round_max_bond:
            h2 = ctypes.c_void_p()
            ctx.synchronize()
            t0 = time.perf_counter()
            nat.call("qtt_tt_round", ctx.handle, y.handle, 1e-8, 0, ctypes.byref(h2))
            tr = time.perf_counter() - t0
            yr = DeviceTrain(h2, ctx)
            out["round"] = {"ms": tr * 1e3, "max_rank": int(max(c.shape[2] for c in yr.cores()))}
        else:
            out["round"] = {"skipped": f"bond rank {16 * r} > {a.round_max_bond} (device SVD limit)"}
        del y
        print(json.dumps(out), flush=True)
        lines.append(out)
    if a.out:
        with open(a.out, "w") as fh:
            for o in lines:
                fh.write(json.dumps(o) + "\n")


if __name__ == "__main__":
    main()
