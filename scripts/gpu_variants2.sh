#!/bin/bash
# parity of each variant library, then k_force timing at c4 2^24 and 2^26 (auto bins)
mkdir -p gpurun_out
TAG=${TAG:-v2}
for L in variants/*.so; do ABSIM_GPU_LIB=$PWD/$L timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_frames.py -m gpu -q -x 2>&1 | tail -1 | sed "s#^#$L #" >> gpurun_out/${TAG}_pytest.log; done
timeout 1200 python scripts/sweep_force.py --config c4 --n 16777216 --libs variants/*.so --bins 0x0 > gpurun_out/${TAG}_sweep_c4_24.log 2>&1
timeout 1200 python scripts/sweep_force.py --config c4 --libs variants/*.so --bins 0x0 > gpurun_out/${TAG}_sweep_c4_26.log 2>&1
tail -n 12 gpurun_out/${TAG}_*.log
