"""Reference fixtures for the TT-cross port: the UNMODIFIED reference
ttfem.cross.cross_interpolate (/root/reference/pkg/src/ttfem/cross.py:273-365) on seeded test
functions; stores the pivot index sets, the sampled-error history, the ranks and the dense
result, which tests/test_gpu_cross.py compares against the device implementation.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cross_golden.py
"""
import os

import numpy as np

import ttfem.cross as rc
import ttfem.tt as rtt

HERE = os.path.dirname(os.path.abspath(__file__))


def case_rank3():
    rng = np.random.default_rng(11)
    dims = (4, 4, 4, 4)
    ranks = [1, 3, 3, 3, 1]
    cores = [rng.standard_normal((ranks[k], dims[k], ranks[k + 1])) for k in range(4)]
    ref = rtt.TensorTrain(cores)
    full = rtt.tt_to_dense(ref).reshape(dims)
    return dims, (lambda idx: full[tuple(np.asarray(idx).T)]), rc.CrossConfig(initial_rank=4), full


def case_smooth():
    # f(i) = 1 / (1 + x) on a QTT grid of 2^10 points, x = i / 2^10 (a smooth, rank-growing case)
    d = 10
    dims = (2,) * d
    w = 2 ** np.arange(d - 1, -1, -1)
    full = 1.0 / (1.0 + (np.arange(2 ** d) / 2 ** d))
    return dims, (lambda idx: full[np.asarray(idx) @ w]), rc.CrossConfig(rel_convergence_tol=1e-10), full.reshape(dims)


def case_reciprocal():
    # reciprocal_tt of a one-signed "Jacobian" 2 + sin on a 4^5 grid
    dims = (4,) * 5
    w = 4 ** np.arange(4, -1, -1)
    v = 2.0 + np.sin(np.arange(4 ** 5) / 37.0)
    return dims, (lambda idx: v[np.asarray(idx) @ w]), rc.CrossConfig(), (1.0 / v).reshape(dims)


def main():
    out = {}
    for name, make in (("rank3", case_rank3), ("smooth", case_smooth), ("recip", case_reciprocal)):
        dims, f, cfg, full = make()
        if name == "recip":
            tt, rep = rc.reciprocal_tt(f, dims, cfg)
        else:
            tt, rep = rc.cross_interpolate(f, dims, cfg)
        out[f"{name}__dense"] = rtt.tt_to_dense(tt)
        out[f"{name}__ranks"] = np.array(tt.ranks)
        out[f"{name}__errors"] = np.array(rep.sampled_errors)
        out[f"{name}__sweeps"] = np.array(rep.sweeps_used)
        out[f"{name}__evaluations"] = np.array(rep.evaluations)
        out[f"{name}__converged"] = np.array(rep.converged)
        out[f"{name}__nbonds"] = np.array(len(rep.left_indices))
        for b, (l, r) in enumerate(zip(rep.left_indices, rep.right_indices)):
            out[f"{name}__left{b}"] = np.asarray(l)
            out[f"{name}__right{b}"] = np.asarray(r)
        print(name, rep.converged, rep.sweeps_used, rep.evaluations, tt.ranks,
              np.linalg.norm(rtt.tt_to_dense(tt) - full.ravel()) / np.linalg.norm(full))
    np.savez_compressed(os.path.join(HERE, "cross_ref.npz"), **out)


if __name__ == "__main__":
    main()
