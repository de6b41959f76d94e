timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_stages.py tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/s4q_tests.log 2>&1; echo rc=$? >> gpurun_out/s4q_tests.log
tools/ab.sh s4q "5:intensity 3:intensity 1:intensity 4:intensity" - var/prev.so
