#!/bin/bash
# round-2 profile evidence for the current build (c4 @ 2^26)
timeout 600 python bench.py --steps 3 --warmup 6 --no-cpu --no-e2e > gpurun_out/r2e_plain.json 2>&1 || exit 1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r2e_launches_c4.csv \
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2e_ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_force -s 8 -c 1 \
  -o gpurun_out/r2e_force_c4 python bench.py --steps 3 --warmup 6 --no-cpu --no-e2e > gpurun_out/r2e_ncu_full.log 2>&1
tail -1 gpurun_out/r2e_ncu_full.log
