#!/bin/bash
# One GPU iteration: detect+describe parity tests, then benches of the headline
# and the dense / single-stream configs.  Usage: tools/gpu_iter.sh TAG [long]
tag=${1:-it}
tests="tests/test_gpu_pipeline.py tests/test_gpu_stages.py tests/test_gpu_configs.py"
[ "$2" = "long" ] && tests="$tests tests/test_gpu_long.py"
timeout 900 python -m pytest $tests -x -q -m gpu > gpurun_out/${tag}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_tests.log
for cm in 5:intensity 5:none 4:intensity 1:intensity; do
  c=${cm%%:*}; m=${cm##*:}
  timeout 300 python bench.py --config $c --mode $m --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --gen cuda \
    > gpurun_out/${tag}_c${c}_${m}.log 2>&1
done
