"""Per-iteration time of the local CG (fused persistent kernel vs per-step launches)
on random SPD local systems of the C2/C3/C5 shapes: python tools/cg_bench.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2501_12151_b200 import _native as nat  # noqa: E402


def spd_local(rl, R, rr, m=2, seed=0):
    rng = np.random.default_rng(seed)
    gl = rng.standard_normal((R, rl, rl))
    phil = np.einsum("aij,akj->iak", gl, gl) / rl + 1e-6 * np.eye(rl)[:, None, :]
    gr = rng.standard_normal((R, rr, rr))
    phir = np.einsum("aij,akj->iak", gr, gr) / rr + 1e-6 * np.eye(rr)[:, None, :]
    G = rng.standard_normal((R, m, m, R)) / R
    A = np.einsum("amnb,apnb->ampb", G, G) + 1e-6 * np.einsum("ab,mn->amnb", np.eye(R), np.eye(m))
    rhs = rng.standard_normal((rl, m, rr))
    prev = rng.standard_normal((rl, m, rr)) * 0.1
    return [nat.f64(a) for a in (phil, A, phir, rhs, prev)]


def main():
    ctx = nat.default_context()
    for rl, R, rr in [(68, 49, 68), (100, 52, 100), (196, 52, 196)]:
        phil, A, phir, rhs, prev = spd_local(rl, R, rr)
        m = 2
        flops = 2.0 * rl * R * rl * m * rr + 2.0 * rl * m * R * R * m * rr + 2.0 * rl * m * rr * R * rr
        for fused in (1, 0):
            u = np.empty((rl, m, rr))
            lam, its = ctypes.c_double(), ctypes.c_int()
            tt = {}
            for cap in (1, 400):
                best = 1e30
                for rep in range(3):
                    t0 = time.perf_counter()
                    nat.call("qtt_local_solve", ctx.handle, nat.dptr(phil), nat.dptr(A), nat.dptr(phir),
                             nat.dptr(rhs), nat.dptr(prev), rl, R, m, R, rr, 1, 0, 1e-300, cap, fused,
                             nat.dptr(u), ctypes.byref(lam), ctypes.byref(its))
                    best = min(best, time.perf_counter() - t0)
                tt[cap] = (best, its.value)
            per = (tt[400][0] - tt[1][0]) / max(1, tt[400][1] - tt[1][1])
            print(f"r={rl} R={R} fused={fused} iters={its.value} us/iter={per * 1e6:.1f} "
                  f"K1 TF/s (whole iteration)={flops / per / 1e12:.2f}", flush=True)


if __name__ == "__main__":
    main()
