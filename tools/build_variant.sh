#!/bin/bash
# Dev tool: build libmpgabor with extra -D flags into paper_2202_12380_b200/libmpgabor_<tag>.so
# for A/B timing (MPGABOR_LIB=<path> python tools/...).  usage: tools/build_variant.sh <tag> -DFOO ...
set -e
cd "$(dirname "$0")/../paper_2202_12380_b200"
tag=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -cudart static "$@" -o libmpgabor_${tag}.so csrc/analysis.cu csrc/mploop.cu csrc/mpmulti.cu csrc/synth.cu csrc/runtime.cu
echo built paper_2202_12380_b200/libmpgabor_${tag}.so
