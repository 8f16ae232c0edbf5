#!/bin/bash
# build library variants in parallel: scripts/build_variants.sh name1 "-DFLAGS..." name2 "-DFLAGS..." ...
cd "$(dirname "$0")/.."
mkdir -p paper_2301_06984_b200/_lib
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  ( /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false $flags \
      -Xcompiler -fPIC -shared -Iinclude -ldl paper_2301_06984_b200/csrc/absim_gpu.cu \
      -o paper_2301_06984_b200/_lib/var_$name.so 2>&1 | grep -E "error|ptxas info.*k_list" ; echo "built $name" ) &
done
wait
