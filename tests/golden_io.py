"""Readers for the frozen reference fixtures in tests/golden (see make_golden.py)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def train(d, name):
    n = int(d[f"{name}__n"])
    return [d[f"{name}__{k}"] for k in range(n)]


def amen_config(d):
    rel, cap = d["cfg_rounding"]
    return {
        "residual_tol": float(d["cfg_residual_tol"]),
        "max_sweeps": int(d["cfg_max_sweeps"]),
        "enrichment_rank": int(d["cfg_enrichment_rank"]),
        "local_solver": str(d["cfg_local_solver"]),
        "direct_dim_cap": int(d["cfg_direct_dim_cap"]),
        "local_iter_cap": int(d["cfg_local_iter_cap"]),
        "rounding": (float(rel), None if cap < 0 else int(cap)),
        "seed": int(d["cfg_seed"]),
        "stagnation_strikes": int(d["cfg_stagnation_strikes"]),
    }


AMEN_CASES = sorted(f for f in os.listdir(GOLDEN) if f.startswith("amen_") and f.endswith(".npz"))


def load_qstep(path):
    """Read a QSTEP1 core-step state file (written by the engine under QTT_DUMP_STEP, or by
    tests/golden/make_headline_step.py): header ints (sweep, core, forward, rank, iters,
    n_in, n_out), scalars (lam_max before the step, ||f||, the step's lam), then the
    n_in input arrays and n_out output arrays, each as int32 dims (3) + float64 data."""
    raw = open(path, "rb").read()
    if raw[:6] != b"QSTEP1":
        raise ValueError(f"{path}: not a QSTEP1 file")
    hdr = np.frombuffer(raw, dtype=np.int32, count=7, offset=6)
    sc = np.frombuffer(raw, dtype=np.float64, count=3, offset=6 + 28)
    off = 6 + 28 + 24
    arrs = []
    for _ in range(int(hdr[5]) + int(hdr[6])):
        d = np.frombuffer(raw, dtype=np.int32, count=3, offset=off)
        off += 12
        n = int(np.prod(d))
        arrs.append(np.frombuffer(raw, dtype=np.float64, count=n, offset=off).reshape(tuple(int(v) for v in d)).copy())
        off += 8 * n
    n_in = int(hdr[5])
    return {"sweep": int(hdr[0]), "core": int(hdr[1]), "forward": bool(hdr[2]), "rank": int(hdr[3]),
            "iters": int(hdr[4]), "lam_max_in": float(sc[0]), "f_norm": float(sc[1]), "lam": float(sc[2]),
            "inputs": arrs[:n_in], "outputs": arrs[n_in:]}


STEP_INPUTS = ("x_k", "x_nb", "z_k", "phi_k", "phi_k1", "phiz_k", "phiz_k1", "psi_k", "psi_k1", "psiz_k", "psiz_k1",
               "A_k", "f_k")
STEP_OUTPUTS = ("x_k", "x_nb", "z_k", "phi", "phiz", "psi", "psiz")


def step_trains(K, A_k, f_k, k):
    """Operator / rhs trains of order K carrying the step's own A_k (R0, m*n, R1) and f_k at
    core k and zero filler elsewhere, rank-chained (core k-1 ends in R0 / r0, core k+1 starts
    with R1 / r1): what qtt_amen_step needs, independent of the host assembly's round-off."""
    R0, mn, R1 = A_k.shape
    m = int(round(mn ** 0.5))
    r0, _, r1 = f_k.shape
    A, f = [], []
    for j in range(K):
        if j == k:
            A.append(A_k.reshape(R0, m, m, R1))
            f.append(f_k)
            continue
        a0 = 1 if j != k + 1 else R1
        a1 = 1 if j != k - 1 else R0
        f0 = 1 if j != k + 1 else r1
        f1 = 1 if j != k - 1 else r0
        n = 3 if j == 0 else 2  # the 3D problems' component core leads (assembly3d.py)
        A.append(np.zeros((a0, n, n, a1)))
        f.append(np.zeros((f0, n, f1)))
    return A, f



def headline_inputs(name):
    """The device-assembled operator and load of a headline config (C3, C5), as committed QTT1
    files under tests/golden/headline/ (tools/headline_dump.py inputs): the reference-side
    scripts solve exactly the system the B200 solved (the device assembly is deterministic;
    host assemblies differ at round-off level)."""
    from paper_2501_12151_b200.serialize import load_tt
    h = os.path.join(GOLDEN, "headline")
    A = load_tt(os.path.join(h, f"{name.lower()}_op.qtt1"))
    f = load_tt(os.path.join(h, f"{name.lower()}_rhs.qtt1"))
    return [np.asarray(c) for c in A.cores], [np.asarray(c) for c in f.cores]
