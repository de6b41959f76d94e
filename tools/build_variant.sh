#!/bin/bash
# Experiment build of the library with extra nvcc flags: tools/build_variant.sh OUT.so [-DFOO=1 ...]
# (select it at run time with VF_LIB=OUT.so)
out=$1; shift
cd "$(dirname "$0")/../paper_1503_06959_b200/csrc" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -shared \
  -cudart static "$@" vf_capi.cu vf_match.cu vf_ransac.cu vf_format.cpp -o "$OLDPWD/$out"
