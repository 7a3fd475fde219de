"""Time the device SVD at the bond widths between the square single-CTA Jacobi (n <= 112)
and the block Jacobi threshold (QTT_BJ_MIN, default 160): python tools/svd_mid.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402

from svd_bench import mat  # noqa: E402
from paper_2501_12151_b200 import _native as nat  # noqa: E402

ctx = nat.default_context()
for m, n in [(232, 116), (256, 128), (280, 140), (318, 159), (392, 196)]:
    a = mat(m, n, 8.0)
    u, s, vt = np.empty((m, n)), np.empty(n), np.empty((n, n))
    best = 1e30
    for rep in range(3):
        t0 = time.perf_counter()
        nat.call("qtt_svd", ctx.handle, nat.dptr(a), m, n, nat.dptr(u), nat.dptr(s), nat.dptr(vt))
        best = min(best, time.perf_counter() - t0)
    err = np.max(np.abs(s - np.linalg.svd(a, compute_uv=False))) / s[0]
    print(f"{m}x{n} ms={best * 1e3:.2f} sv_err={err:.1e}", flush=True)
