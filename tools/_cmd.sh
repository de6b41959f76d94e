timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_stages.py tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/s4i_tests.log 2>&1; echo rc=$? >> gpurun_out/s4i_tests.log
run() { name=$1; shift; for cm in 5:intensity 4:intensity 3:intensity 2:intensity 1:intensity 5:none; do c=${cm%%:*}; m=${cm##*:}
env "$@" timeout 300 python bench.py --config $c --mode $m --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --gen cuda > gpurun_out/s4i_${name}_c${c}_${m}.log 2>&1
done; }
run unfused VF_NMS_FUSED=0
run fused VF_NMS_FUSED=1
run unfused2 VF_NMS_FUSED=0
run fused2 VF_NMS_FUSED=1
