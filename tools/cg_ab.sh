#!/bin/bash
# A/B runs of tools/cg_iter_bench.py under different engine knobs: tools/cg_ab.sh "shapes" "ENV1" "ENV2" ...
shapes=$1; shift
for e in "$@"; do
  echo "== $e"
  env $e python tools/cg_iter_bench.py $shapes 2>&1 | grep -E "^r=" 
done
