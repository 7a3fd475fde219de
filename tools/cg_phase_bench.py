"""Per-iteration phase times of the fused CG kernel (device globaltimer, QTT_DEBUG)
on random SPD local systems: python tools/cg_phase_bench.py [rl,R,rr ...]
Tile/compose choices can be forced with QTT_CG_TILE_A, QTT_CG_TILE_3, QTT_CG_COMPOSE."""
import ctypes
import os
import re
import sys
import tempfile

os.environ.setdefault("QTT_DEBUG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2501_12151_b200 import _native as nat  # noqa: E402
from cg_bench import spd_local  # noqa: E402

LINE = re.compile(r"cg_fused dims (\d+),(\d+),(\d+) R (\d+) S3 (\d+) tiles (\d+),(\d+) composed (\d) grid (\d+) "
                  r"iters (\d+): ns step1 (\d+) step2 (\d+) step3 (\d+) red (\d+) upd (\d+) pupd (\d+)")


def main():
    shapes = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]] or \
        [(40, 52, 40), (68, 49, 68), (100, 52, 100), (104, 52, 108), (196, 52, 196)]
    ctx = nat.default_context()
    tmp = tempfile.TemporaryFile(mode="w+")
    saved = os.dup(2)
    os.dup2(tmp.fileno(), 2)
    try:
        for rl, R, rr in shapes:
            phil, A, phir, rhs, prev = spd_local(rl, R, rr)
            u = np.empty((rl, 2, rr))
            lam, its = ctypes.c_double(), ctypes.c_int()
            for rep in range(6):
                nat.call("qtt_local_solve", ctx.handle, nat.dptr(phil), nat.dptr(A), nat.dptr(phir),
                         nat.dptr(rhs), nat.dptr(prev), rl, R, 2, R, rr, 1, 0, 1e-300, 400, 1,
                         nat.dptr(u), ctypes.byref(lam), ctypes.byref(its))
    finally:
        os.dup2(saved, 2)
    tmp.seek(0)
    rows = {}
    for line in tmp:
        if ("per-CTA" in line or "cta_dump" in line or "timeline" in line) and os.environ.get("QTT_SHOW_CTA"):
            print(line.strip())
        m = LINE.search(line)
        if m:
            v = [int(g) for g in m.groups()]
            rows.setdefault(tuple(v[:3]), []).append(v)
    names = ["step1", "step2", "step3", "red", "upd", "pupd"]
    for key, vs in rows.items():
        vs = vs[1:]  # first call: module/attribute warm-up
        it = vs[0][9]
        per = np.median(np.array([v[10:16] for v in vs], dtype=float), axis=0) / max(1, it) / 1e3
        rl, m, rr = key
        R = vs[0][3]
        flops = 2.0 * rl * R * rl * m * rr + 2.0 * rl * m * R * R * m * rr + 2.0 * rl * m * rr * R * rr
        tot = per.sum()
        print(f"r={rl},{rr} R={R} S3={vs[0][4]} tiles={vs[0][5]},{vs[0][6]} composed={vs[0][7]} iters={it} "
              + " ".join(f"{n}={p:.1f}" for n, p in zip(names, per))
              + f" total={tot:.1f}us K1-alg TF/s={flops / (tot * 1e-6) / 1e12:.2f}", flush=True)


if __name__ == "__main__":
    main()
