#!/bin/bash
mkdir -p gpurun_out
for w in C1 C2; do
  timeout 900 python tools/run_config.py $w > gpurun_out/run_$w.json 2> gpurun_out/run_$w.err; echo "$w rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/run_$w.json')); print({k: d[k] for k in ('workload','dof','op_ranks_max','gpu_s','converged','sweeps','final','max_rank')})"
done
timeout 1200 python tools/run_config.py C5 --max-sweeps 8 > gpurun_out/run_C5.json 2> gpurun_out/run_C5.err; echo "C5 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/run_C5.json')); print({k: d[k] for k in ('workload','dof','op_ranks_max','gpu_s','converged','sweeps','final','max_rank')}, d['res_hist'])"
tail -3 gpurun_out/run_C5.err
