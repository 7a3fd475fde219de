#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.log
QTT_DEBUG=1 timeout 600 python tools/qr_bench.py 10406,5203 8192,4096 > gpurun_out/qr.log 2>&1; echo "qr rc=$?"
grep -v "ms: panel" gpurun_out/qr.log | tail -4
grep "ms: panel" gpurun_out/qr.log | tail -3
timeout 600 python tools/cert_bench.py C3 2>&1 | tail -2
