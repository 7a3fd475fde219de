import hashlib, json, sys, numpy as np
sys.path.insert(0, '.')
from paper_2501_12151_b200.configs import WORKLOADS, build
out = {}
for n in sys.argv[1:]:
    prob, _, _ = build(WORKLOADS[n])
    h = hashlib.sha256()
    for c in prob.op + prob.rhs:
        h.update(np.ascontiguousarray(c).tobytes())
    out[n] = {"sha": h.hexdigest()[:16], "op_ranks": list(prob.op_ranks)}
print(json.dumps(out))
