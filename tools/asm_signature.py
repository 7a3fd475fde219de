import sys, time, json, hashlib, numpy as np
sys.path.insert(0, '.')
from paper_2501_12151_b200.configs import WORKLOADS, build
for n in sys.argv[1:]:
    t0 = time.perf_counter(); prob, _, _ = build(WORKLOADS[n]); dt = time.perf_counter() - t0
    h = hashlib.sha256()
    for c in prob.op + prob.rhs: h.update(np.ascontiguousarray(c).tobytes())
    print(json.dumps({n: {"sha": h.hexdigest()[:16], "s": round(dt, 2), "op_ranks": list(prob.op_ranks)}}), flush=True)
