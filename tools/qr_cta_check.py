"""Device QR (qtt_qr) vs numpy.linalg.qr on sweep-shaped matrices, and its time per call
(QTT_QR_CTA=0 selects the unblocked single-CTA kernel for A/B)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2501_12151_b200 import _native as nat  # noqa: E402


def main():
    ctx = nat.default_context()
    rng = np.random.default_rng(0)
    for m, n in [(200, 100), (208, 104), (100, 100), (200, 104), (8, 4), (16, 20), (33, 17), (136, 68),
                 (104, 208), (1, 5), (5, 1), (392, 50), (250, 40)]:
        a = rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 10.0)
        k = min(m, n)
        q, r = np.empty((m, k)), np.empty((k, n))
        nat.call("qtt_qr", ctx.handle, nat.dptr(a), m, n, nat.dptr(q), nat.dptr(r))
        qn, rn = np.linalg.qr(a)
        eq = np.linalg.norm(q - qn) / np.sqrt(k)
        er = np.linalg.norm(r - rn) / np.linalg.norm(rn)
        t0 = time.perf_counter()
        for _ in range(20):
            nat.call("qtt_qr", ctx.handle, nat.dptr(a), m, n, nat.dptr(q), nat.dptr(r))
        dt = (time.perf_counter() - t0) / 20
        print(f"{m}x{n}: |Q-Qnp| {eq:.2e} |R-Rnp|/|R| {er:.2e}  {dt * 1e6:.0f} us/call (incl. H2D/D2H)")


if __name__ == "__main__":
    main()
