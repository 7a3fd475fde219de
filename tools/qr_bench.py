"""Blocked Householder QR at certification / rounding sizes:
    QTT_DEBUG=2 python tools/qr_bench.py [m,n ...]
QTT_DEBUG>=1 prints the per-stage times of geqrf_blocked; >=2 the panel timeline per column."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2501_12151_b200 import _native as nat  # noqa: E402

shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(10406, 5203), (8192, 4096)]
ctx = nat.default_context()
for m, n in shapes:
    a = np.random.default_rng(0).standard_normal((m, n))
    k = min(m, n)
    r = np.empty((k, n))
    for rep in range(2):
        t0 = time.perf_counter()
        nat.call("qtt_qr", ctx.handle, nat.dptr(a), m, n, None, nat.dptr(r))
        print(f"qr {m}x{n} (R only) {time.perf_counter() - t0:.3f} s", flush=True)
