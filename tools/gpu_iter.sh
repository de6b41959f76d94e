#!/bin/bash
# One GPU iteration: detect+describe parity tests, then the default bench
# (no CPU baseline / e2e).  Usage: tools/gpu_iter.sh TAG
tag=${1:-it}
timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_stages.py tests/test_gpu_configs.py -x -q \
  > gpurun_out/${tag}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench.log 2>&1
