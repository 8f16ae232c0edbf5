#!/bin/bash
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_c4.json 2> gpurun_out/r2a_c4.err || { tail -5 gpurun_out/r2a_c4.err; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r2a_launches_c4.csv python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2a_ncu.log 2>&1
