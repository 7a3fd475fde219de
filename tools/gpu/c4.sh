#!/bin/bash
# Config-4 parity tests + microbench on the GPU.
mkdir -p gpurun_out
python -m pytest tests/test_c4.py -q -m gpu > gpurun_out/c4_tests.log 2>&1; echo "c4 tests rc=$?"
tail -3 gpurun_out/c4_tests.log
timeout 900 python tools/c4_bench.py --out gpurun_out/c4_bench.jsonl > gpurun_out/c4_bench.log 2>&1; echo "c4 bench rc=$?"
cat gpurun_out/c4_bench.log | tail -8
# one full ncu capture of the persistent CG kernel at full rank (C3 sweep ~25, dims 96x2x98)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cg_tma -s 258 -c 1 \
    -o gpurun_out/cg_tma_full python tools/run_config.py C3 --max-sweeps 26 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
