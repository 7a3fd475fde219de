"""Direct local solve (dense local matrix + fused Cholesky, amen.py:181-191) on random SPD
local systems of the C3 shapes: QTT_DEBUG=1 python tools/chol_bench.py  (prints the fused
kernel's phase times per call)."""
import ctypes
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
import numpy as np  # noqa: E402

from cg_bench import spd_local  # noqa: E402
from paper_2501_12151_b200 import _native as nat  # noqa: E402


def main():
    ctx = nat.default_context()
    for rl, R, rr in [(16, 46, 16), (24, 50, 24), (32, 51, 32), (44, 52, 44), (32, 52, 64)]:
        phil, A, phir, rhs, prev = spd_local(rl, R, rr)
        m = 2
        dim = rl * m * rr
        u = np.empty((rl, m, rr))
        lam, its = ctypes.c_double(), ctypes.c_int()
        best = 1e30
        for rep in range(3):
            t0 = time.perf_counter()
            nat.call("qtt_local_solve", ctx.handle, nat.dptr(phil), nat.dptr(A), nat.dptr(phir),
                     nat.dptr(rhs), nat.dptr(prev), rl, R, m, R, rr, 0, 4096, 1e-6, 400, 1,
                     nat.dptr(u), ctypes.byref(lam), ctypes.byref(its))
            best = min(best, time.perf_counter() - t0)
        print(f"dim {dim} ({rl},{m},{rr}) R={R}: {best * 1e3:.3f} ms wall (incl. H2D/D2H), "
              f"chol {dim ** 3 / 3 / 1e9:.2f} GFLOP", flush=True)


if __name__ == "__main__":
    main()
