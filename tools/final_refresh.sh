#!/bin/bash
# Evidence pass 1 of a round's final kernels (one GPU): ncu launch lists of one
# step per workload, then `ncu --set full` reports of the main kernels of the
# headline (config 5) and the dense (config 4) step.  Pass 2 is tools/bench_all.sh
# after tools/traffic_json.py has turned the launch lists into profiles/*.json
# (bench.py reads the step's DRAM traffic from there).   tools/final_refresh.sh TAG
tag=${1:-fin}
tools/prof_all.sh ${tag}p 5:intensity 5:none 5:binning 4:intensity 4:none 3:intensity 2:intensity 1:intensity
for k in k_desc_fused k_fast k_nms_test k_pyr_o k_sat k_propagate; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:^$k -c 1 -f \
    -o gpurun_out/${tag}full5_$k python tools/prof_step.py --config 5 --mode intensity --warmup 3 \
    > gpurun_out/${tag}full5_$k.out 2>&1
done
for k in k_desc_fused k_nms_test k_fast; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:^$k -c 1 -f \
    -o gpurun_out/${tag}full4_$k python tools/prof_step.py --config 4 --mode intensity --warmup 3 \
    > gpurun_out/${tag}full4_$k.out 2>&1
done
