#!/bin/bash
# Config-4 parity tests + microbench on the GPU.
mkdir -p gpurun_out
python -m pytest tests/test_c4.py -q -m gpu > gpurun_out/c4_tests.log 2>&1; echo "c4 tests rc=$?"
tail -3 gpurun_out/c4_tests.log
timeout 900 python tools/c4_bench.py --out gpurun_out/c4_bench.jsonl > gpurun_out/c4_bench.log 2>&1; echo "c4 bench rc=$?"
cat gpurun_out/c4_bench.log | tail -8
