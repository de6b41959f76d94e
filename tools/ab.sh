#!/bin/bash
# A/B of library variants on one box: tools/ab.sh TAG "config:mode ..." lib1.so lib2.so ...  ("-" = the in-tree library)
tag=$1; cms=$2; shift 2
for rep in 1 2; do
for lib in "$@"; do
  for cm in $cms; do
    c=${cm%%:*}; m=${cm##*:}
    name=$(basename ${lib%.so})
    if [ "$lib" = "-" ]; then unset VF_LIB; name=base; else export VF_LIB=$PWD/$lib; fi
    timeout 300 python bench.py --config $c --mode $m --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --gen cuda \
      > gpurun_out/${tag}_${name}_c${c}_${m}_r${rep}.log 2>&1
  done
done
done
unset VF_LIB
