"""Benchmark: QTT AMEn time-to-solution on the BASELINE.json headline workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C3]

One *step* is one complete ``amen_solve`` of the workload (BASELINE.json metric:
"time-to-solution at 2^30 cells; local-matvec FP64 TFLOP/s vs peak" -> config C3:
clamped unit cube, 2^10 nodes per axis = 1023^3 cells ~ 2^30, 3.2e9 DOF, tol 1e-6,
max rank 96).  ``value`` is the solve time with A, f, x0 already resident in HBM
(device handles), CUDA events on the engine stream, L2 flushed before every step;
``e2e`` is the same solve through the public Python API (``amen_solve`` with numpy
host cores in, numpy cores out), H2D/D2H included.  The path does not shard
(replicas only): under torchrun every rank solves its own replica,
the reported time is the max over ranks.

``--impl reference`` times the CPU oracle (oracle/qtt_oracle.py, the restatement of
the reference ttfem path) on this host by a bounded sample, extrapolated over the
recorded trajectory of the solve (oracle/cpu_baseline.py); rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peaks_r01.jsonl")
TRAJ_DIR = os.path.join(ROOT, "profiles")


def fp64_peak():
    """Measured FP64 tensor (DMMA) peak on this pool's B200 (tools/fp64_peak.cu)."""
    best = None
    if os.path.exists(FP64_PEAK_FILE):
        for line in open(FP64_PEAK_FILE):
            d = json.loads(line)
            if d.get("what") == "dmma_m8n8k4":
                best = max(best or 0.0, d["tflops"])
    return (best, "measured DMMA m8n8k4 peak, profiles/fp64_peaks_r01.jsonl") if best else \
        (40.0, "fallback nominal B200 FP64 tensor")


def k1_traffic():
    """DRAM bytes per K1 call inside the CG kernel, from the committed ncu --set full capture
    (profiles/r02/cg_tma_traffic.json; the operands stay L2-resident across iterations)."""
    p = os.path.join(ROOT, "profiles", "r02", "cg_tma_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d["dram_bytes_per_k1"], f"DRAM bytes per K1 call at {d['shape']}, {d['source']}"


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if os.environ.get("BENCH_BACKEND", "nccl") == "nccl" else "gloo"
        dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, v, local):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for i, name in enumerate(names):
                if len(r) > 5 + i and "Active" in r[5 + i] and "Not" not in r[5 + i]:
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def build_problem(name):
    from paper_2501_12151_b200.configs import WORKLOADS, build
    w = WORKLOADS[name]
    t0 = time.perf_counter()
    prob, x0, kw = build(w)
    return w, prob, x0, kw, time.perf_counter() - t0


def amen_config(kw):
    from paper_2501_12151_b200.amen import AmenConfig
    from paper_2501_12151_b200.tt import TruncationPolicy
    kw = dict(kw)
    rel, cap = kw.pop("rounding")
    return AmenConfig(rounding=TruncationPolicy(rel, cap), **kw)


def workload_config(w, extra=None):
    cfg = {"workload": f"{w.name}: 3D Q1 elasticity, clamped unit cube, 2^{w.L} nodes/axis "
                       f"({w.cells_per_axis}^3 cells), {w.dof:.3g} DOF, serial-binary QTT, "
                       f"tol {w.tol:g}, max rank {w.max_rank}, x0 rank-2 N(0,1) seed 0, AmenConfig seed 2024",
           "cells": w.cells_per_axis ** 3, "dof": w.dof, "tol": w.tol, "max_rank": w.max_rank,
           "max_sweeps": w.max_sweeps, "l2": "flushed (256 MiB write) before every timed step"}
    if extra:
        cfg.update(extra)
    return cfg


def cert_shapes(A_cores, x_cores, f_cores):
    """(rows, cols) of the QR/SVD unfoldings in the reference's certification sweep."""
    K = len(A_cores)
    R = [1] + [c.shape[3] for c in A_cores]
    r = [1] + [c.shape[2] for c in x_cores]
    rf = [1] + [c.shape[2] for c in f_cores]
    tot = [R[k] * r[k] + (rf[k] if 0 < k < K else 0) for k in range(K + 1)]
    tot[0] = tot[K] = 1
    shapes, right = [], 1
    for k in range(K - 1, 0, -1):
        m = A_cores[k].shape[1]
        rows = m * right
        right = min(tot[k], rows)
        shapes.append((rows, tot[k]))
    return shapes


def source_digest():
    """sha256 over the engine sources (csrc/*.cu, *.cuh): identifies the build whose recorded
    trajectory the CPU arm extrapolates over (a kernel change can move the trajectory)."""
    import glob
    import hashlib
    h = hashlib.sha256()
    for f in sorted(glob.glob(os.path.join(ROOT, "paper_2501_12151_b200", "csrc", "*.cu*"))):
        h.update(os.path.basename(f).encode())
        h.update(open(f, "rb").read())
    return h.hexdigest()


def cpu_baseline(trace, n_cert, shapes, sweeps, budget):
    from oracle import cpu_baseline as CB
    tables, info = CB.sample_rates(budget_s=budget)
    parts = CB.extrapolate_parts(trace, tables, n_cert=n_cert, cert_shapes=shapes)
    secs = parts["total_s"]
    return secs, {
        "breakdown_s": {k: round(v, 2) for k, v in parts.items()},
        "cores": CB.host_cores(), "kind": "port",
        "sample": (f"oracle primitives (local matvec, env update, dense+Cholesky, SVD/QR) timed on this host at "
                   f"ranks {info['ranks']} and dense dims {info['dense_dims']} in {info['sample_s']:.1f} s plus one "
                   f"certification-size {info['cert_unfolding']} in {info['cert_sample_s']:.1f} s, "
                   f"extrapolated over the solve's recorded trajectory ({len(trace)} local solves, "
                   f"{int(sum(int(t[10]) for t in trace))} CG iterations, {sweeps} sweeps, {n_cert} certifications)"),
    }


def run_reference(args, world, rank):
    """CPU arm: the oracle restatement of the reference path, bounded sample."""
    if rank != 0:
        return
    name = args.workload
    w, prob, x0, kw, _ = build_problem(name)
    path = os.path.join(TRAJ_DIR, f"trajectory_{name}.json")
    if not os.path.exists(path):
        print(json.dumps({"impl": "reference", "unavailable": f"no recorded trajectory {path}"}))
        return
    traj = json.load(open(path))
    if traj.get("source_sha256") != source_digest():
        # the recorded trajectory belongs to another build of the engine: refuse to extrapolate
        print(json.dumps({"impl": "reference", "unavailable": f"{path} was recorded by another engine build "
                          "(source digest mismatch); re-record it with bench.py"}))
        return
    trace = np.array(traj["trace"], dtype=np.int64)
    x_ranks = traj["x_ranks"]
    xc = [np.zeros((x_ranks[k], prob.dims[k], x_ranks[k + 1])) for k in range(len(prob.dims))]
    shapes = cert_shapes(prob.op, xc, prob.rhs)
    from oracle import cpu_baseline as CB
    for _ in range(args.warmup):  # warm numpy/OpenBLAS thread pools
        CB.sample_rates(ranks=(8,), dense_dims=(256,), budget_s=1.0)
    times = []
    info = None
    for _ in range(max(1, args.steps)):
        secs, info = cpu_baseline(trace, traj["certifications"], shapes, traj["sweeps"],
                                  budget=max(10.0, min(25.0, 150.0 / max(1, args.steps))))
        times.append(secs)
    v = float(np.mean(times))
    line = {"metric": "time-to-solution at 2^30 cells (C3 QTT AMEn solve)", "value": v, "unit": "s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference", "config": workload_config(w),
            "cpu_baseline": dict(info, value=v, unit="s"),
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def c4_summary(ctx, ranks=(128, 256), reps=2):
    """Config 4 (BASELINE.json configs[3]) K1/K2 sweep at the two largest ranks: one right-env
    pre-pass + one L->R sweep of local matvecs and env updates on resident random TT data
    (configs.c4_problem, seed 1), per-launch-group CUDA events; see tools/c4_bench.py."""
    from paper_2501_12151_b200 import kernels
    from paper_2501_12151_b200.configs import c4_problem
    from paper_2501_12151_b200.tt import DeviceTrain
    peak, _ = fp64_peak()
    out = {}
    for r in ranks:
        op, x = c4_problem(r)
        dA, dx = DeviceTrain.upload(op, ctx), DeviceTrain.upload(x, ctx)
        kernels.matvec_sweep(dA, dx, ctx=ctx, timing=True, split_timing=True, return_y=False)
        ts = []
        for _ in range(reps):
            ctx.flush_l2()
            ts.append(kernels.matvec_sweep(dA, dx, ctx=ctx, timing=True, split_timing=True, return_y=False)[1])
        k1 = min(t["k1_ms"] for t in ts)
        k2 = min(t["k2_ms"] for t in ts)
        sw = min(t["sweep_ms"] for t in ts)
        t = ts[0]
        out[f"r{r}"] = {"sweep_ms": sw, "k1_tflops": t["k1_flops"] / k1 / 1e9,
                        "k1_frac": t["k1_flops"] / k1 / 1e9 / peak, "k2_tflops": t["k2_flops"] / k2 / 1e9,
                        "sweep_tflops": (t["k1_flops"] + t["k2_flops"]) / sw / 1e9}
        del dA, dx
    return out


def run_ours(args, world, rank, local):
    import torch

    from paper_2501_12151_b200 import _native as nat
    from paper_2501_12151_b200.amen import amen_solve, amen_solve_device, random_draws
    from paper_2501_12151_b200.tt import DeviceTrain, TensorTrain, TTLinearOperator

    torch.cuda.set_device(local)
    w, prob, x0, kw, t_asm = build_problem(args.workload)
    cfg = amen_config(kw)
    ctx = nat.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    A, f, X0 = TTLinearOperator(prob.op), TensorTrain(prob.rhs), TensorTrain(x0)
    draws = random_draws(A, f.dims, cfg)
    dA, df, dx0 = (DeviceTrain.upload(t.cores, ctx) for t in (A, f, X0))
    K = A.order

    def solve_resident():
        return amen_solve_device(dA, df, dx0, cfg, draws, K, ctx)

    for _ in range(args.warmup):
        _, winfo = solve_resident()
        if os.environ.get("BENCH_VERBOSE"):
            print(f"warmup solve: {winfo['sweeps_used']} sweeps, {winfo['final_relative_residual']!r}",
                  file=sys.stderr, flush=True)
    ctx.synchronize()

    ctx.set_profiling(True)  # deferred CUDA events around every K1/K2 launch (no syncs)
    ctx.reset_stats()
    launches0 = nat.launch_count()
    times, info = [], None
    trace_from = 0
    with ClockSampler(local) as clk:
        for step in range(args.steps):
            if step == args.steps - 1:  # the trajectory (cpu_baseline, trajectory file) is ONE solve's
                trace_from = len(ctx.trace())
            ctx.flush_l2()
            barrier(world)
            ctx.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dx, info = solve_resident()
            e1.record(stream)
            ctx.synchronize()
            torch.cuda.synchronize(local)
            barrier(world)
            times.append(e0.elapsed_time(e1) / 1e3)
    launches = nat.launch_count() - launches0
    stats = ctx.stats()
    trace = ctx.trace()[trace_from:]
    ctx.set_profiling(False)
    x_ranks = [1] + [int(c.shape[2]) for c in dx.cores()]
    value = max_over_ranks(world, float(np.mean(times)), local)

    # e2e through the public API: numpy cores in (pinned copies H2D), numpy cores out
    e2e_times = []
    h2d = sum(c.nbytes for t in (A, f, X0) for c in t.cores) + draws.nbytes
    d2h = 0
    for _ in range(max(1, args.e2e_steps)):
        ctx.flush_l2()
        barrier(world)
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        x, rep = amen_solve(A, f, X0, cfg, ctx=ctx)
        e1.record(stream)
        ctx.synchronize()
        torch.cuda.synchronize(local)
        e2e_times.append(e0.elapsed_time(e1) / 1e3)
        d2h = sum(c.nbytes for c in x.cores) + 8 * (2 + cfg.max_sweeps * (K + 2))
    e2e = max_over_ranks(world, float(np.mean(e2e_times)), local)

    k1_tf = stats["k1_timed_flops"] / stats["k1_ms"] / 1e9 if stats["k1_ms"] > 0 else 0.0
    peak, peak_src = fp64_peak()
    steps = max(1, args.steps)
    roofline = {
        "bound": "tensor",
        "kernel": "K1 local matvec: inside the persistent TMA/DMMA CG kernel (cg_tma_kernel; %globaltimer spans "
                  "of its matvec phases incl. the split-K reduction) and the DMMA GEMM chain elsewhere (CUDA events)",
        "achieved": k1_tf, "peak": peak, "unit": "TFLOP/s", "frac": k1_tf / peak,
        "peak_source": peak_src,
        "per_launch": {"calls_per_step": stats["k1_calls"] / steps,
                       "avg_flops": stats["k1_timed_flops"] / max(1, stats["k1_calls"]),
                       "avg_us": 1e3 * stats["k1_ms"] / max(1, stats["k1_calls"])},
        "share_of_step": stats["k1_ms"] / 1e3 / max(1e-9, sum(times)),
        "env_update_tflops": stats["env_timed_flops"] / stats["env_ms"] / 1e9 if stats["env_ms"] > 0 else None,
        "traffic": None,
    }
    tr = k1_traffic()
    if tr is not None:
        roofline["traffic"], roofline["traffic_source"] = tr
    line = {"metric": "time-to-solution at 2^30 cells (C3 QTT AMEn solve)", "value": value, "unit": "s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(w),
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU", "assembly_s": round(t_asm, 2),
            "result": {"converged": info["converged"], "sweeps": info["sweeps_used"],
                       "final_relative_residual": info["final_relative_residual"], "max_rank": max(x_ranks),
                       "cg_iterations": int(stats["cg_iters"] / steps),
                       "sweeps_per_s": info["sweeps_used"] / value},
            "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "roofline": roofline}
    if rank == 0:
        line["clocks"] = clk.summary()
        traj = {"workload": args.workload, "source_sha256": source_digest(), "trace": trace.tolist(),
                "x_ranks": x_ranks, "cg_iterations": int(trace[:, 10].sum()),
                "certifications": int(stats["certifications"] / steps), "sweeps": info["sweeps_used"]}
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        json.dump(traj, open(os.path.join(ROOT, "gpurun_out", f"trajectory_{args.workload}.json"), "w"))
        if world == 1 and not args.no_c4:
            line["c4_microbench"] = c4_summary(ctx)
        if world == 1 and not args.no_cpu:
            shapes = cert_shapes(prob.op, dx.cores(), prob.rhs)
            secs, cb = cpu_baseline(trace, traj["certifications"], shapes, info["sweeps_used"], budget=20.0)
            line["cpu_baseline"] = dict(cb, value=secs, unit="s")
        print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-c4", action="store_true", help="skip the config-4 K1 sweep summary")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
