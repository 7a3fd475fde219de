"""CPU baseline of the QTT AMEn solve by a bounded sample -- TEST/BENCH INFRASTRUCTURE.

Used only by ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``).  A full
reference solve of config C3 (2^30 cells) takes hours on host cores, so
the time-to-solution is *extrapolated*:

1. the oracle's own primitives (local matvec, environment update, dense local
   matrix + Cholesky, SVD/QR of the sweep unfoldings; oracle/qtt_oracle.py, which
   restates ttfem/amen.py and ttfem/tt.py) are timed on this host at a handful of
   shapes of the workload -- the bounded sample, ~10-30 s of CPU work;
2. their flop rates are interpolated (log-log in problem size) and summed over the
   solve's recorded trajectory: every local solve of the run (sweep, core, ranks,
   local path, CG iterations), as recorded by the device engine on the same
   inputs (same algorithm and stopping rules), plus the certification checks.

numpy/scipy use all host threads (OpenBLAS), so this port is *faster* per flop than
the reference, whose einsum contractions run on one core: the baseline is generous
to the CPU side.
"""
from __future__ import annotations

import math
import os
import time

import numpy as np
import scipy.linalg

from . import qtt_oracle as O


def host_cores() -> int:
    return os.cpu_count() or 1


def _time_base(fn, min_time=0.05, max_reps=20):
    fn()  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        fn()
        reps += 1
        el = time.perf_counter() - t0
        if el >= min_time or reps >= max_reps:
            return el / reps


def k1_flops(rl, R0, m, R1, rr):
    return 2.0 * rl * R0 * rl * m * rr + 2.0 * rl * m * R1 * R0 * m * rr + 2.0 * rl * m * rr * R1 * rr


def env_flops(rl, R0, m, R1, rr):
    return k1_flops(rl, R0, m, R1, rr)


class RateTable:
    """Measured GFLOP/s of one primitive at a few sizes; log-log interpolation."""

    def __init__(self):
        self.pts = []  # (log flops, rate flops/s)

    def add(self, flops, seconds):
        self.pts.append((math.log(max(flops, 1.0)), flops / max(seconds, 1e-9)))
        self.pts.sort()

    def rate(self, flops):
        lf = math.log(max(flops, 1.0))
        xs = [p[0] for p in self.pts]
        ys = [math.log(p[1]) for p in self.pts]
        if lf <= xs[0]:
            return math.exp(ys[0])
        if lf >= xs[-1]:
            return math.exp(ys[-1])
        return math.exp(float(np.interp(lf, xs, ys)))

    def seconds(self, flops):
        return flops / self.rate(flops)


_CERT_SAMPLE = []


def _cert_size_sample(rows=8192, cols=4096):
    """One SVD and one QR of a rows x cols unfolding (cached for the process)."""
    if not _CERT_SAMPLE:
        big = np.random.default_rng(7).standard_normal((rows, cols))
        t0 = time.perf_counter()
        np.linalg.svd(big, full_matrices=False)
        t1 = time.perf_counter()
        np.linalg.qr(big)
        t2 = time.perf_counter()
        _CERT_SAMPLE.extend([("svd", 14.0 * rows * cols * cols, t1 - t0), ("qr", 4.0 * rows * cols * cols, t2 - t1)])
    return list(_CERT_SAMPLE)


def sample_rates(R=52, m=2, ranks=(8, 16, 24, 32, 48, 64, 80, 100, 112),
                 dense_dims=(256, 512, 1024, 2048, 2304, 3200, 4096), seed=0, budget_s=15.0):
    """Time the oracle primitives at representative shapes (the bounded sample, about
    budget_s of host work: every measurement repeats for ~budget_s / 60)."""
    rng = np.random.default_rng(seed)
    t_start = time.perf_counter()
    mt = max(0.05, budget_s / 60.0)

    def _time(fn, min_time=None, max_reps=200):
        return _time_base(fn, min_time=mt if min_time is None else min_time, max_reps=max_reps)

    tables = {k: RateTable() for k in ("k1", "env", "dense", "chol", "svd", "qr")}
    shapes = []
    for i, r in enumerate(ranks):
        if i > 0 and time.perf_counter() - t_start > budget_s:
            break
        phil = rng.standard_normal((r, R, r))
        phir = rng.standard_normal((r, R, r))
        A = rng.standard_normal((R, m, m, R))
        x = rng.standard_normal((r, m, r))
        fl = k1_flops(r, R, m, R, r)
        tables["k1"].add(fl, _time(lambda: O.local_matvec(phil, A, phir, x)))
        tables["env"].add(fl, _time(lambda: O.env_left(phil, x, A, x)))
        mat = rng.standard_normal((2 * r, r))
        tables["svd"].add(14.0 * (2 * r) * r * r, _time(lambda: np.linalg.svd(mat, full_matrices=False)))
        aug = rng.standard_normal((2 * r, r + 4))
        tables["qr"].add(4.0 * (2 * r) * (r + 4) ** 2, _time(lambda: np.linalg.qr(aug)))
        shapes.append(r)
    # large unfoldings, the size class of the certification sweeps: 2048 x 1024 every call,
    # plus one real certification-size 8192 x 4096 SVD and QR (timed once per process: ~20-60 s
    # of host work; C3's certification unfoldings are up to ~10400 x 5200)
    big = rng.standard_normal((2048, 1024))
    tables["svd"].add(14.0 * 2048 * 1024 * 1024, _time(lambda: np.linalg.svd(big, full_matrices=False),
                                                        max_reps=3))
    tables["qr"].add(4.0 * 2048 * 1024 * 1024, _time(lambda: np.linalg.qr(big), max_reps=3))
    t_cert = time.perf_counter()
    for name, fl, sec in _cert_size_sample():  # (its own ~20-60 s, outside the sample budget)
        tables[name].add(fl, sec)
    cert_s = time.perf_counter() - t_cert
    t_start += cert_s
    for i, d in enumerate(dense_dims):
        if i > 0 and time.perf_counter() - t_start > budget_s:
            break
        rl = int(round(math.sqrt(d / m)))
        phil = rng.standard_normal((rl, R, rl))
        phir = rng.standard_normal((rl, R, rl))
        A = rng.standard_normal((R, m, m, R))
        fl = 2.0 * rl * rl * R * m * m * R + 2.0 * (rl * m * rl) ** 2 * R
        tables["dense"].add(fl, _time(lambda: O.local_dense(phil, A, phir), max_reps=10))
        g = rng.standard_normal((d, d))
        spd = g @ g.T + d * np.eye(d)
        b = rng.standard_normal(d)

        def chol():
            c = scipy.linalg.cho_factor(spd, lower=True)
            scipy.linalg.cho_solve(c, b)
            float(np.abs(spd).sum(axis=1).max())

        tables["chol"].add(d ** 3 / 3.0, _time(chol, max_reps=10))
    return tables, {"ranks": shapes, "dense_dims": list(dense_dims),
                    "cert_unfolding": "8192 x 4096 SVD + QR", "cert_sample_s": cert_s,
                    "sample_s": time.perf_counter() - t_start}


def extrapolate(trace, tables, n_cert=0, cert_shapes=None):
    """Seconds the oracle would need for the recorded trajectory (see extrapolate_parts)."""
    return extrapolate_parts(trace, tables, n_cert, cert_shapes)["total_s"]


def extrapolate_parts(trace, tables, n_cert=0, cert_shapes=None):
    """Seconds the oracle would need for the recorded trajectory, split into the sweep work
    and the certifications.

    ``total_s`` follows the reference's certification (amen.py:87-99: tt_round of the
    rank R*r + r_f difference train at 0.1*tol -- a QR sweep plus an SVD sweep -- then
    tt_norm); ``like_for_like_s`` replaces it by what the device does, the exact QR-sweep
    norm of the unrounded difference train (one QR per bond).

    trace: rows (sweep, core, rl, m, rr, zl, zr, R0, R1, path, iters) -- one per local
    solve.  Per core step the reference does: 1 local rhs, the local solve (dense
    build + Cholesky, or iters+1 local matvecs), 2 mixed residuals (2 local
    matvecs), an SVD and two QRs of the unfoldings, 4 environment updates.
    """
    total = 0.0
    cert = cert_ll = 0.0
    for row in trace:
        _, _, rl, m, rr, zl, zr, R0, R1, path, iters = (int(v) for v in row)
        k1 = k1_flops(rl, R0, m, R1, rr)
        if path == 0:
            dim = rl * m * rr
            dense = 2.0 * rl * rl * R0 * m * m * R1 + 2.0 * dim * dim * R1
            total += tables["dense"].seconds(dense) + tables["chol"].seconds(dim ** 3 / 3.0)
        else:
            total += (iters + 1) * tables["k1"].seconds(k1)
        total += 2 * tables["k1"].seconds(k1 * max(zl, rl) / max(rl, 1))  # mixed residuals
        rows, cols = rl * m, rr
        k = min(rows, cols)
        total += tables["svd"].seconds(14.0 * max(rows, cols) * k * k)
        total += tables["qr"].seconds(4.0 * rows * (k + 4) ** 2) * 2
        total += 2 * tables["env"].seconds(k1) + 2 * tables["env"].seconds(k1 * zl / max(rl, 1))
    # certifications: tt_round + tt_norm QR/SVD sweeps over the rank R*r + r_f train
    if n_cert and cert_shapes:
        per = per_ll = 0.0
        for (rows, cols) in cert_shapes:
            per += tables["svd"].seconds(14.0 * rows * cols * min(rows, cols))
            per += 2 * tables["qr"].seconds(4.0 * rows * cols * min(rows, cols))
            per_ll += tables["qr"].seconds(4.0 * rows * cols * min(rows, cols))
        cert, cert_ll = n_cert * per, n_cert * per_ll
    return {"total_s": total + cert, "sweeps_s": total, "certification_s": cert,
            "like_for_like_s": total + cert_ll, "certification_like_for_like_s": cert_ll}
