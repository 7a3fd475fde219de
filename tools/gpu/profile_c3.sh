#!/bin/bash
# C3 phase profile + ncu launch list + one full capture of the CG kernel (round-1 evidence).
set -x
mkdir -p gpurun_out
python tools/run_config.py C3 --profile > gpurun_out/c3_profile.json 2> gpurun_out/c3_profile.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3_s12.csv python tools/run_config.py C3 --max-sweeps 12 > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cg_tma -s 150 -c 1 \
    -o gpurun_out/cg_tma_full python tools/run_config.py C3 --max-sweeps 12 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
