#!/bin/bash
# parity of the group force kernel + LPA sweep on c4
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/lpa_tests.log 2>&1
tail -5 gpurun_out/lpa_tests.log
timeout 900 python scripts/sweep_force.py --config c4 --n 16777216 --bins 2x2 --lpas 1 2 4 8 16 32 > gpurun_out/lpa_sweep24.log 2>&1
timeout 900 python scripts/sweep_force.py --config c4 --bins 2x2 --lpas 1 4 8 16 > gpurun_out/lpa_sweep26.log 2>&1
