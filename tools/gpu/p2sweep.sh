#!/bin/bash
for p in "" "13,13,74" "13,9,50" "13,5,29" "7,25,74" "13,25,148" "13,7,30" "13,7,45"; do
  if [ -z "$p" ]; then echo "default"; QTT_DEBUG=1 python tools/cg_iter_bench.py 100,52 2>&1 | tail -1 | cut -c1-160;
  else echo "P2=$p"; QTT_TMA_P2=$p QTT_DEBUG=1 python tools/cg_iter_bench.py 100,52 2>&1 | tail -1 | cut -c1-160; fi
done
for p in "9,13" "5,13" "18,10" "9,7"; do
  echo "P1=$p"; QTT_TMA_P1=$p QTT_DEBUG=1 python tools/cg_iter_bench.py 100,52 2>&1 | tail -1 | cut -c1-160
done
