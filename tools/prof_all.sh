#!/bin/bash
# ncu launch lists (duration + DRAM bytes + SM throughput + warp instructions) of one step per workload.
# Usage: tools/prof_all.sh TAG "config:mode ..."
tag=${1:-p}; shift
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
for cm in ${@:-"5:intensity 5:none 4:intensity 1:intensity"}; do
  c=${cm%%:*}; m=${cm##*:}
  timeout 600 ncu --profile-from-start off --clock-control none --metrics $M --csv \
    --log-file gpurun_out/${tag}_c${c}_${m}.csv python tools/prof_step.py --config $c --mode $m --warmup 3 \
    > gpurun_out/${tag}_c${c}_${m}.out 2>&1
done
