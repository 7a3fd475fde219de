"""Per-iteration phase times of the persistent TMA CG kernel on random SPD local
systems of the C3 shapes (R = 52, r = 24..100):

    QTT_DEBUG=1 python tools/cg_iter_bench.py [r,R ...]

With QTT_DEBUG=1 the library prints, per solve, the in-kernel %globaltimer spans of
the four phases summed over the iterations ("cg_fused dims ... ns step1 .. upd ..");
this tool converts them to microseconds per iteration and adds the K1 TFLOP/s of
the matvec part (phases 1+2+reduction) and of the whole iteration."""
import ctypes
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

LINE = re.compile(r"cg_fused dims (\d+),(\d+),(\d+) R (\d+) S3 (\d+) tiles (\d+),(\d+) composed (\d) grid (\d+) "
                  r"iters (\d+): ns step1 (\d+) step2 (\d+) step3 (\d+) red (\d+) upd (\d+) pupd (\d+)")


def child(shapes):
    import numpy as np

    from cg_bench import spd_local
    from paper_2501_12151_b200 import _native as nat
    ctx = nat.default_context()
    for rl, R in shapes:
        rr = rl
        phil, A, phir, rhs, prev = spd_local(rl, R, rr)
        m = 2
        u = np.empty((rl, m, rr))
        lam, its = ctypes.c_double(), ctypes.c_int()
        for rep in range(3):
            nat.call("qtt_local_solve", ctx.handle, nat.dptr(phil), nat.dptr(A), nat.dptr(phir),
                     nat.dptr(rhs), nat.dptr(prev), rl, R, m, R, rr, 1, 0, 1e-300, 400, 1,
                     nat.dptr(u), ctypes.byref(lam), ctypes.byref(its))
        print(f"done {rl} {R} {its.value}", flush=True)


def main():
    shapes = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]] or \
        [(24, 52), (32, 52), (48, 52), (64, 52), (80, 52), (100, 52)]
    if os.environ.get("_CG_ITER_CHILD"):
        child(shapes)
        return
    env = dict(os.environ, QTT_DEBUG=os.environ.get("QTT_DEBUG", "1"), _CG_ITER_CHILD="1")
    p = subprocess.run([sys.executable, __file__] + [f"{a},{b}" for a, b in shapes], env=env,
                       capture_output=True, text=True)
    sys.stderr.write(p.stderr[-2000:] if p.returncode else "")
    last = {}
    for line in p.stderr.splitlines():
        mm = LINE.search(line)
        if mm:
            v = [int(g) for g in mm.groups()]
            last[(v[0], v[3])] = v
    for (rl, R), v in sorted(last.items()):
        it = max(1, v[9])
        ph = [x / it / 1e3 for x in v[10:16]]
        m, rr = 2, rl
        flops = 2.0 * rl * R * rl * m * rr + 2.0 * rl * m * R * R * m * rr + 2.0 * rl * m * rr * R * rr
        # cg_tma marks: slot 1 phase 1, 2 phase 2, 3 split-K reduce + p.q, 4 x/r/z update
        print(f"r={rl} R={R} S3={v[4]} tiles={v[5]},{v[6]} iters={it}: us/iter phase1 {ph[1]:.2f} phase2 {ph[2]:.2f} "
              f"reduce {ph[3]:.2f} update {ph[4]:.2f} | K1 {flops / 1e6:.0f} MFLOP, "
              f"K1 TF/s (p1+p2+reduce) {flops / ((ph[1] + ph[2] + ph[3]) * 1e-6) / 1e12:.2f}, "
              f"whole-iteration TF/s {flops / (sum(ph) * 1e-6) / 1e12:.2f}", flush=True)
    if not last:
        print(p.stdout, p.stderr[-3000:])


if __name__ == "__main__":
    main()
