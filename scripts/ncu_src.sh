#!/bin/bash
# source-attributed profile of the per-lane force kernel (c4 @ 2^24)
export ABSIM_LPA=${ABSIM_LPA:-1}
timeout 600 python bench.py --agents 16777216 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/src_plain.json 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_force -s 3 -c 1 \
  -o gpurun_out/r2_force_src python bench.py --agents 16777216 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/src_ncu.log 2>&1
tail -3 gpurun_out/src_ncu.log
