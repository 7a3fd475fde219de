#!/bin/bash
# ncu launch list (time + DRAM bytes per launch) of the first 16 C3 sweeps: ranks reach the
# full 100 by sweep ~10, so the persistent CG kernel carries its full-rank share.
mkdir -p gpurun_out
timeout 1700 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3_s16.csv python tools/run_config.py C3 --max-sweeps 16 > gpurun_out/ncu_list16.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py list gpurun_out/launches_c3_s16.csv | head -30
gzip -kf gpurun_out/launches_c3_s16.csv
