#!/bin/bash
# Round-2 evidence at HEAD: GPU tests, one full ncu capture of the CG kernel at the C3 full-rank
# shape, and the ncu launch list of the first 12 C3 sweeps.
mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/gputest_r02.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cg_tma -s 150 -c 1 \
    -o gpurun_out/cg_tma_full_r02 python tools/run_config.py C3 --max-sweeps 12 > gpurun_out/ncu_full_r02.log 2>&1
echo "ncu full rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3_s12_r02.csv python tools/run_config.py C3 --max-sweeps 12 > gpurun_out/ncu_list_r02.log 2>&1
echo "ncu list rc=$?"
python tools/ncu_summary.py list gpurun_out/launches_c3_s12_r02.csv > gpurun_out/launches_c3_s12_r02_summary.txt 2>&1
gzip -f gpurun_out/launches_c3_s12_r02.csv
tail -3 gpurun_out/gputest_r02.log
