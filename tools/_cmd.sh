for c in 2 1 3 4 5; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/s4o_bench_c$c.log 2>&1; done
