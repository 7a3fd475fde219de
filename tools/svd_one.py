import sys, ctypes
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import numpy as np
from svd_bench import mat
from paper_2501_12151_b200 import _native as nat
ctx = nat.default_context()
for m, n in [(200, 100), (208, 104)]:
    a = mat(m, n, 5.0)
    k = min(m, n)
    u, s, vt = np.empty((m, k)), np.empty(k), np.empty((k, n))
    for rep in range(2):
        nat.call("qtt_svd", ctx.handle, nat.dptr(a), m, n, nat.dptr(u), nat.dptr(s), nat.dptr(vt))
