#!/bin/sh
# Fast register / spill check of the non-template kernels of pdcs_kernels.cuh
# (one small TU, ~10 s, no library link):  tools/kcheck.sh [sed-expression] [kernel-regex]
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
T=/tmp/pdcs_kcheck
rm -rf $T && mkdir -p $T/include $T/pkg/csrc
cp $R/include/pdcs.h $T/include/
cp $R/paper_2603_15504_b200/csrc/*.cuh $T/pkg/csrc/
if [ -n "$1" ]; then sed -i "$1" $T/pkg/csrc/pdcs_kernels.cuh; fi
printf '#include <cstdint>\n#include "pdcs_kernels.cuh"\n' > $T/pkg/csrc/t.cu
cd $T/pkg/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -cubin \
  -o t.cubin t.cu -Xptxas -v 2>&1 | grep -A3 "Compiling entry.*${2:-.}" | grep -v "^--" | \
  sed -e 's/ptxas info    : //' | c++filt
