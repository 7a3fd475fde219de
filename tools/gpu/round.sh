#!/bin/bash
mkdir -p gpurun_out
export QTT_DEBUG_JACOBI=1
timeout 900 python -m pytest tests/test_gpu_tt.py tests/test_c4.py -q -m gpu -x > gpurun_out/round_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/round_tests.log
QTT_DEBUG=1 timeout 900 python tools/c4_bench.py --round-max-bond 4096 --reps 2 --out gpurun_out/c4_bench2.jsonl > gpurun_out/c4_bench2.log 2>&1; echo "c4 bench rc=$?"
grep "tt_round" gpurun_out/c4_bench2.log
grep "block jacobi" gpurun_out/c4_bench2.log | sort | uniq -c | sort -rn | head -12
grep "geqrf" gpurun_out/c4_bench2.log | sort | uniq -c | sort -rn | head -12
python -c "
import json
for l in open('gpurun_out/c4_bench2.jsonl'):
    d=json.loads(l); print(d['r'], 'apply', round(d['apply']['ms'],2), 'ms', round(d['apply']['gbs']), 'GB/s', 'round', d['round'])
"
