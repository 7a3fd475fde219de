import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2501_12151_b200 import _native as nat
ctx = nat.default_context()
a = np.random.default_rng(0).standard_normal((200, 100))
q, r = np.empty((200, 100)), np.empty((100, 100))
for _ in range(2):
    nat.call("qtt_qr", ctx.handle, nat.dptr(a), 200, 100, nat.dptr(q), nat.dptr(r))
