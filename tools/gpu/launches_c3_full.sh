#!/bin/bash
# ncu launch list (kernel time only) of the whole C3 solve (bench workload), for the kernel
# shares of the step; per-launch times are serialised and cold-cache.
mkdir -p gpurun_out
timeout 2700 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3_full.csv python tools/run_config.py C3 > gpurun_out/ncu_full_list.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py list gpurun_out/launches_c3_full.csv > gpurun_out/launches_c3_full_summary.txt 2>&1
head -30 gpurun_out/launches_c3_full_summary.txt
gzip -kf gpurun_out/launches_c3_full.csv
