"""Time the exact certification sweep (residual_norm) at C2/C3 ranks."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2501_12151_b200 import _native as nat  # noqa: E402
from paper_2501_12151_b200.configs import WORKLOADS, build  # noqa: E402
from paper_2501_12151_b200.tt import DeviceTrain  # noqa: E402

for name in sys.argv[1:]:
    prob, _, _ = build(WORKLOADS[name])
    ctx = nat.default_context()
    rng = np.random.default_rng(0)
    dims = prob.dims
    K = len(dims)
    for r in (100,):
        ranks = [1] + [min(r, 2 ** min(k, K - k)) for k in range(1, K)] + [1]
        x = [rng.standard_normal((ranks[k], dims[k], ranks[k + 1])) / np.sqrt(ranks[k]) for k in range(K)]
        dA, dx, df = (DeviceTrain.upload(t, ctx) for t in (prob.op, x, prob.rhs))
        out, used = ctypes.c_double(), ctypes.c_int()
        for rep in range(2):
            t0 = time.perf_counter()
            nat.call("qtt_residual_norm", ctx.handle, dA.handle, dx.handle, df.handle, 0, ctypes.byref(out),
                     ctypes.byref(used))
            print(name, r, "exact", out.value, f"{time.perf_counter() - t0:.3f} s", flush=True)
