"""State-injected single core step at the headline shapes.

Input: a core-step state the device engine dumped in the middle of a full solve
(QTT_DUMP_STEP=sweep,core,path; tools/headline_dump.py on the B200): environments
phi/phiz/psi/psiz at both bonds, x_k, its neighbour, z_k, the running lam_max and ||f||,
plus the engine's own outputs of that step.  Here the UNMODIFIED reference primitives run the
same step -- the per-core body of ttfem.amen._sweep (/root/reference/pkg/src/ttfem/amen.py:
324-365, forward direction), every arithmetic call a reference function:
_local_rhs, _solve_local (dense Cholesky or SciPy CG), _mixed_residual, _truncated_factor,
numpy.linalg.qr, _phi_left_step, _psi_left_step.  The output fixture (QSTEP1: the device's
inputs + the REFERENCE outputs, lam, truncation rank and CG iteration count) is checked by
tests/test_gpu_headline.py, which re-runs the step through qtt_amen_step on the GPU.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_headline_step.py DUMP OUT CFG
"""
from __future__ import annotations

import json
import os
import struct
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import ttfem.amen as ram  # noqa: E402
import ttfem.tt as rtt  # noqa: E402

rtt._ALLOWED_MODES = (2, 3, 4, 8, 9)

from paper_2501_12151_b200.configs import WORKLOADS, build  # noqa: E402
from tests.golden_io import load_qstep  # noqa: E402


def write_qstep(path, hdr, sc, arrays_in, arrays_out):
    with open(path, "wb") as fh:
        fh.write(b"QSTEP1")
        fh.write(struct.pack("<7i", *hdr))
        fh.write(struct.pack("<3d", *sc))
        for a in list(arrays_in) + list(arrays_out):
            a3 = np.ascontiguousarray(a, dtype="<f8").reshape(a.shape + (1,) * (3 - a.ndim))
            fh.write(struct.pack("<3i", *a3.shape))
            fh.write(a3.tobytes())


def main(dump, out, cfg_name):
    st = load_qstep(dump)
    assert st["forward"], "forward steps only"
    prob, _, kw = build(WORKLOADS[cfg_name], rounding="host")
    rel, cap = kw.pop("rounding")
    cfg = ram.AmenConfig(rounding=rtt.TruncationPolicy(rel, cap), **kw)
    k, K = st["core"], len(prob.op)
    x_k, x_nb, z_k, phi_k, phi_k1, phiz_k, phiz_k1, psi_k, psi_k1, psiz_k, psiz_k1, a3, fc = st["inputs"]
    m = x_k.shape[1]
    ac = a3.reshape(a3.shape[0], m, m, a3.shape[2])  # the device's own A_k and f_k (dumped with the state)
    asm = {"A_k_vs_host_assembly": float(np.abs(ac - prob.op[k]).max()) if ac.shape == prob.op[k].shape else
           f"shapes differ: device {ac.shape} host {prob.op[k].shape}"}
    psi_k, psi_k1, psiz_k, psiz_k1 = (a[:, :, 0] for a in (psi_k, psi_k1, psiz_k, psiz_k1))
    rl, m, rr = x_k.shape

    calls = [0]
    base = ram._local_matvec

    def counted(*a):
        calls[0] += 1
        return base(*a)

    t0 = time.time()
    # ---- amen.py:324-365, forward branch, the reference's own primitives
    rhs = ram._local_rhs(psi_k, fc, psi_k1)
    ram._local_matvec = counted
    try:
        u, lam = ram._solve_local(phi_k, ac, phi_k1, rhs, x_k, cfg, st["sweep"], k)
    finally:
        ram._local_matvec = base
    dim = rhs.size
    # matvec calls of the CG branch: SciPy's LinearOperator probes the dtype with one call, cg
    # computes r = b - A x0 with one more when x0 != 0, then one per iteration
    iters = 0 if dim <= cfg.direct_dim_cap else calls[0] - 1 - (1 if np.any(x_k) else 0)
    lam_max = max(st["lam_max_in"], lam)
    delta_abs = cfg.residual_tol * st["f_norm"] / (lam_max * np.sqrt(K - 1))
    zeta = ram._mixed_residual(psiz_k, fc, psiz_k1, phiz_k, ac, u, phiz_k1)
    enrich = ram._mixed_residual(psi_k, fc, psiz_k1, phi_k, ac, u, phiz_k1)
    qfac, w = ram._truncated_factor(u.reshape(rl * m, rr), cfg.rounding, delta_abs)
    aug = np.hstack([qfac, enrich.reshape(rl * m, -1)])
    q, r = np.linalg.qr(aug)
    new_xk = q.reshape(rl, m, q.shape[1])
    absorb = r[:, : qfac.shape[1]] @ w
    new_nb = np.einsum("ab,bnc->anc", absorb, x_nb)
    zq, _ = np.linalg.qr(zeta.reshape(zeta.shape[0] * m, -1))
    new_zk = zq.reshape(zeta.shape[0], m, zq.shape[1])
    phi_new = ram._phi_left_step(phi_k, new_xk, ac, new_xk)
    psi_new = ram._psi_left_step(psi_k, new_xk, fc)
    phiz_new = ram._phi_left_step(phiz_k, new_zk, ac, new_xk)
    psiz_new = ram._psi_left_step(psiz_k, new_zk, fc)
    secs = time.time() - t0
    rank = qfac.shape[1]
    write_qstep(out, (st["sweep"], k, 1, rank, iters, len(st["inputs"]), 7), (st["lam_max_in"], st["f_norm"], lam),
                st["inputs"], [new_xk, new_nb, new_zk, phi_new, phiz_new, psi_new, psiz_new])
    # how far the device's own in-solve outputs are from the reference's (informational)
    dev = st["outputs"]
    sup_ref = np.einsum("anb,bmc->anmc", new_xk, new_nb)
    sup_dev = np.einsum("anb,bmc->anmc", dev[0], dev[1])
    summ = {"config": cfg_name, "sweep": st["sweep"], "core": k, "dim": int(dim), "reference_s": secs,
            "ref_rank": int(rank), "dev_rank": st["rank"], "ref_lam": lam, "dev_lam": st["lam"],
            "ref_cg_iters": int(iters), "dev_cg_iters": st["iters"],
            "u_supercore_rel": float(np.linalg.norm(sup_dev - sup_ref) / np.linalg.norm(sup_ref)), **asm}
    json.dump(summ, open(out + ".json", "w"), indent=1)
    print(summ)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
