#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f32_tests.log 2>&1
tail -3 gpurun_out/f32_tests.log
for f in 1 0; do ABSIM_F32=$f timeout 600 python scripts/sweep_force.py --config c4 --n 16777216 --bins 2x2 > gpurun_out/f32_$f.log 2>&1; done
ABSIM_F32=1 timeout 600 python scripts/sweep_force.py --config c4 --bins 2x2 > gpurun_out/f32_1_26.log 2>&1
