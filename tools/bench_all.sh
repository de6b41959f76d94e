#!/bin/bash
# Every BASELINE config through bench.py (one GPU).  Usage: tools/bench_all.sh TAG [K]
tag=${1:-all}; K=${2:-30}
for c in 1 2 3 4 5; do
  timeout 600 python bench.py --config $c --steps $K --warmup 5 --no-cpu-baseline > gpurun_out/${tag}_c${c}.log 2>&1
done
for m in none binning; do
  timeout 600 python bench.py --config 5 --mode $m --steps $K --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c5_${m}.log 2>&1
done
timeout 600 python bench.py --config 4 --mode none --steps $K --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c4_none.log 2>&1
