#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/gpu_tests.log
QTT_DEBUG_JACOBI=1 QTT_DEBUG=1 timeout 900 python tools/c4_bench.py --round-max-bond 4096 --reps 3 --out gpurun_out/c4_bench.jsonl > gpurun_out/c4_bench.log 2>&1; echo "c4 bench rc=$?"
grep "tt_round" gpurun_out/c4_bench.log
grep "block jacobi 4096" gpurun_out/c4_bench.log | head -2
python -c "
import json
for l in open('gpurun_out/c4_bench.jsonl'):
    d=json.loads(l); print(d['r'], 'K1 %.2f TF/s (%.3f)' % (d['sweep']['k1_tflops'], d['sweep']['k1_frac_fp64_peak']), 'apply %.2f ms %.0f GB/s' % (d['apply']['ms'], d['apply']['gbs']), 'round', d['round'])
"
