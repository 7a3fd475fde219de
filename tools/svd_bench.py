"""Time the device SVD (QR + one-sided Jacobi) on truncation-like matrices:
python tools/svd_bench.py   (QTT_DEBUG_JACOBI=1 prints the sweep counts)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2501_12151_b200 import _native as nat  # noqa: E402


def mat(m, n, decay, seed=0):
    rng = np.random.default_rng(seed)
    k = min(m, n)
    u, _ = np.linalg.qr(rng.standard_normal((m, k)))
    v, _ = np.linalg.qr(rng.standard_normal((n, k)))
    s = np.exp(-decay * np.arange(k) / k)
    return nat.f64((u * s) @ v.T)


def main():
    ctx = nat.default_context()
    for m, n in [(200, 100), (100, 200), (208, 104), (136, 68), (392, 196)]:
        for decay in (5.0, 30.0):
            a = mat(m, n, decay)
            k = min(m, n)
            u, s, vt = np.empty((m, k)), np.empty(k), np.empty((k, n))
            best = 1e30
            for rep in range(5):
                t0 = time.perf_counter()
                nat.call("qtt_svd", ctx.handle, nat.dptr(a), m, n, nat.dptr(u), nat.dptr(s), nat.dptr(vt))
                best = min(best, time.perf_counter() - t0)
            ref = np.linalg.svd(a, compute_uv=False)
            err = np.max(np.abs(s - ref) / ref[0])
            rec = np.linalg.norm((u * s) @ vt - a) / np.linalg.norm(a)
            print(f"{m}x{n} decay={decay} ms={best * 1e3:.3f} sv_err={err:.1e} recon={rec:.1e}", flush=True)


if __name__ == "__main__":
    main()


def qr_times():
    ctx = nat.default_context()
    for m, n in [(200, 100), (100, 100), (208, 104)]:
        a = mat(m, n, 5.0)
        q, r = np.empty((m, n)), np.empty((n, n))
        best = 1e30
        for rep in range(5):
            t0 = time.perf_counter()
            nat.call("qtt_qr", ctx.handle, nat.dptr(a), m, n, nat.dptr(q), nat.dptr(r))
            best = min(best, time.perf_counter() - t0)
        print(f"qr {m}x{n} ms={best * 1e3:.3f}", flush=True)


if os.environ.get("QR_TIMES"):
    qr_times()
