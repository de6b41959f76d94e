timeout 900 python -m pytest tests/test_gpu_stages.py -x -q -m gpu -k "three_steps or pipelined" > gpurun_out/s4r_tests.log 2>&1; echo rc=$? >> gpurun_out/s4r_tests.log
python __graft_entry__.py --smoke > gpurun_out/s4r_smoke.log 2>&1; echo rc=$? >> gpurun_out/s4r_smoke.log
timeout 600 python bench.py > gpurun_out/s4r_bench_default.log 2>&1; echo rc=$? >> gpurun_out/s4r_bench_default.log
