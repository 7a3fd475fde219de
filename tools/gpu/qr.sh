#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tt.py tests/test_c4.py -q -m gpu > gpurun_out/round_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/round_tests.log
QTT_DEBUG=2 timeout 600 python tools/qr_bench.py 10406,5203 8192,4096 > gpurun_out/qr.log 2>&1; echo "qr rc=$?"
grep -v "ms: panel" gpurun_out/qr.log | tail -8
grep "ms: panel" gpurun_out/qr.log | tail -2
