#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-v3}
for L in variants/*.so; do ABSIM_GPU_LIB=$PWD/$L timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1 | sed "s#^#$L #" >> gpurun_out/${TAG}_pytest.log; done
for rep in 1 2; do
timeout 1200 python scripts/sweep_force.py --config c4 --libs variants/*.so --bins 0x0 >> gpurun_out/${TAG}_sweep_c4_26.log 2>&1
done
timeout 1200 python scripts/sweep_force.py --config c4 --n 16777216 --libs variants/*.so --bins 0x0 > gpurun_out/${TAG}_sweep_c4_24.log 2>&1
tail -n 12 gpurun_out/${TAG}_*.log
