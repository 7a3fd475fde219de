import sys, os, json, time
sys.path.insert(0, '.')
os.environ["QTT_DEBUG"] = "1"
import numpy as np
from paper_2501_12151_b200 import _native as nat
from paper_2501_12151_b200.configs import WORKLOADS, build
from paper_2501_12151_b200.tt import DeviceTrain, TensorTrain, TTLinearOperator, tt_round
import ctypes
for name in sys.argv[1:]:
    w = WORKLOADS[name]
    prob, x0, kw = build(w)
    ctx = nat.default_context()
    rng = np.random.default_rng(0)
    dims = prob.dims
    K = len(dims)
    for r in (40, 100):
        ranks = [1] + [min(r, 2 ** min(k, K - k)) for k in range(1, K)] + [1]
        x = [rng.standard_normal((ranks[k], dims[k], ranks[k + 1])) / np.sqrt(ranks[k]) for k in range(K)]
        dA, dx, df = DeviceTrain.upload(prob.op, ctx), DeviceTrain.upload(x, ctx), DeviceTrain.upload(prob.rhs, ctx)
        out, used = ctypes.c_double(), ctypes.c_int()
        t0 = time.time()
        nat.call("qtt_residual_norm", ctx.handle, dA.handle, dx.handle, df.handle, 0, ctypes.byref(out), ctypes.byref(used))
        t1 = time.time()
        print(name, r, "gram", out.value, used.value, t1 - t0, flush=True)
        if r > 40: continue
        out2 = ctypes.c_double()
        nat.call("qtt_residual_norm", ctx.handle, dA.handle, dx.handle, df.handle, 1, ctypes.byref(out2), ctypes.byref(used))
        t2 = time.time()
        print(name, r, "gram", out.value, used.value, t1 - t0, "exact", out2.value, t2 - t1, flush=True)
