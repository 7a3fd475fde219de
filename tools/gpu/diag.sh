#!/bin/bash
mkdir -p gpurun_out
export QTT_DEBUG_JACOBI=1
timeout 900 python -m pytest tests/test_gpu_tt.py tests/test_c4.py -q -m gpu -x > gpurun_out/round_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/round_tests.log
QTT_DEBUG=1 timeout 900 python tools/c4_bench.py --ranks 64,256 --round-max-bond 4096 --reps 2 --out gpurun_out/c4_bench3.jsonl > gpurun_out/c4_bench3.log 2>&1; echo "c4 bench rc=$?"
grep "tt_round" gpurun_out/c4_bench3.log
grep "block jacobi 4096" gpurun_out/c4_bench3.log | head -3
grep "block jacobi 1024" gpurun_out/c4_bench3.log | head -2
QTT_DEBUG=1 timeout 600 python tools/cert_bench.py C3 > gpurun_out/cert.log 2>&1; echo "cert rc=$?"
grep -v "^\[qtt\] geqrf" gpurun_out/cert.log | tail -5
grep "^\[qtt\] geqrf" gpurun_out/cert.log | awk '{print $3}' | sort | uniq -c | head -30
python - <<'PY'
import re
tot=[0.0]*5
for l in open('gpurun_out/cert.log'):
    m=re.search(r"geqrf (\d+)x(\d+) ms: panel ([\d.]+) v\+gram\+T ([\d.]+) Y1 ([\d.]+) Y2 ([\d.]+) update ([\d.]+)", l)
    if m:
        for i in range(5): tot[i]+=float(m.group(3+i))
print("geqrf totals over both cert calls (ms): panel %.1f vgramT %.1f Y1 %.1f Y2 %.1f update %.1f" % tuple(tot))
PY
QTT_DEBUG=1 timeout 600 python tools/cg_iter_bench.py > gpurun_out/cg_iter.log 2>&1; echo "cg_iter rc=$?"
cat gpurun_out/cg_iter.log | tail -8
