#!/bin/bash
# Debug library: every launch of the step is followed by cudaDeviceSynchronize
# and an error check naming the kernel (DBG_SYNC), CUDA graphs off.  Used in
# place of compute-sanitizer (closed on the GPU pool):
#   tools/debug_build.sh && VF_LIB=build/dbg.so python -m pytest tests -m gpu
set -e
cd "$(dirname "$0")/../paper_1503_06959_b200/csrc"
mkdir -p ../../build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -DVF_DEBUG -Xcompiler -fPIC -shared \
  -cudart static vf_capi.cu vf_match.cu vf_ransac.cu vf_format.cpp -o ../../build/dbg.so
