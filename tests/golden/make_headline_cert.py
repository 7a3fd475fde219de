"""Independent certification of the GPU's headline solutions.

The device's C3 and C5 solutions (tools/headline_dump.py on the B200, saved as QTT1 under
tests/golden/headline/) are certified here, in the build container, by the reference:

  * C3: the UNMODIFIED reference, ttfem.amen.residual_norm(A, x, f)
    (/root/reference/pkg/src/ttfem/amen.py:87-99 -> tt_apply(policy=None), tt_sub, tt_norm,
    tt.py:330-371, 434-449), and ttfem's own QTT1 reader (serialize.py) loads x.
    Peak host memory ~40 GB (the rank-5201 difference train is materialised twice).
  * C5: the reference path does not fit this host's 62 GB (the rank-10193 difference train
    is ~45 GB, materialised twice), so oracle.qtt_oracle.residual_norm_streaming -- the same
    cores and QR sweep, one core at a time -- certifies it; that streaming restatement is
    itself checked against the unmodified reference on C3 (both values are stored).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_headline_cert.py

writes tests/golden/headline/cert.json; tests/test_gpu_headline.py asserts the device's
certification of the same x equals it to 1e-10 relative.
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import ttfem.amen as ram  # noqa: E402
import ttfem.serialize as rser  # noqa: E402
import ttfem.tt as rtt  # noqa: E402

rtt._ALLOWED_MODES = (2, 3, 4, 8, 9)

from oracle import qtt_oracle as O  # noqa: E402

OUT = os.path.join(HERE, "headline", "cert.json")


def main(which):
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in which:
        # the reference's own QTT1 reader (serialize.py) loads the B200's operator, load and solution
        x = rser.load_tt(os.path.join(HERE, "headline", f"{name.lower()}_x.qtt1"))
        A = rser.load_tt(os.path.join(HERE, "headline", f"{name.lower()}_op.qtt1"))
        f = rser.load_tt(os.path.join(HERE, "headline", f"{name.lower()}_rhs.qtt1"))
        d = {"x_ranks": list(map(int, x.ranks)), "op_ranks": list(map(int, A.ranks))}
        t0 = time.time()
        d["streaming"] = O.residual_norm_streaming(list(A.cores), list(x.cores), list(f.cores))
        d["streaming_s"] = time.time() - t0
        if name == "C3":
            t0 = time.time()
            d["reference"] = float(ram.residual_norm(A, x, f))
            d["reference_s"] = time.time() - t0
        res[name] = d
        json.dump(res, open(OUT, "w"), indent=1)
        print(name, d, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C3", "C5"])
