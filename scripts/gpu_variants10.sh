#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-v10}
for L in variants/*.so; do ABSIM_GPU_LIB=$PWD/$L timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x 2>&1 | tail -1 | sed "s#^#$L #" >> gpurun_out/${TAG}_pytest.log; done
for rep in 1 2; do timeout 1500 python scripts/sweep_force.py --config c4 --libs variants/*.so --bins 0x0 --steps 8 >> gpurun_out/${TAG}_c4.log 2>&1; done
cat gpurun_out/${TAG}_pytest.log; grep -h force_ms gpurun_out/${TAG}_c4.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['lib'], round(d['ms_per_step'],4), round(d['force_ms'],4))"
