#!/bin/bash
# Round-2 state at HEAD: full GPU tests, the bench line, C1/C2/C5 runs and the C4 microbench.
mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/gputest_r02.log 2>&1
tail -3 gpurun_out/gputest_r02.log
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc=$?"
( time python bench.py --impl reference --steps 1 --warmup 1 ) > gpurun_out/bench_r02_reference.json 2> gpurun_out/bench_r02_reference.err; echo "reference arm rc=$?"
for w in C1 C2 C5; do
  timeout 900 python tools/run_config.py $w --profile > gpurun_out/run_$w.json 2> gpurun_out/run_$w.err; echo "$w rc=$?"
done
python tools/c4_bench.py > gpurun_out/c4_bench_r02.jsonl 2> gpurun_out/c4_bench_r02.err; echo "c4 rc=$?"
