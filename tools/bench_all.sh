#!/bin/bash
# Every BASELINE config through bench.py (one GPU), then ncu launch lists of one
# step per config (skipped with a third argument "noprof").  Usage: tools/bench_all.sh TAG [K] [noprof]
tag=${1:-all}; K=${2:-30}
for c in 5 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps $K --warmup 5 > gpurun_out/${tag}_c${c}.log 2>&1
done
for m in none binning; do
  timeout 600 python bench.py --config 5 --mode $m --steps $K --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c5_${m}.log 2>&1
done
timeout 600 python bench.py --config 4 --mode none --steps $K --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c4_none.log 2>&1
timeout 900 python bench.py --impl reference --config 5 --steps 10 --warmup 2 > gpurun_out/${tag}_ref_c5.log 2>&1
[ "$3" = "noprof" ] || tools/prof_all.sh ${tag}p 5:intensity 5:none 5:binning 4:intensity 3:intensity 2:intensity 1:intensity
