tools/bench_all.sh r2x 30 noprof
timeout 1800 python -m pytest tests -q -m gpu -v > gpurun_out/r2x_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2x_gpu_tests.log
