#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-v8}
for rep in 1 2; do
timeout 900 python scripts/sweep_force.py --config c3 --libs variants/*.so --bins 0x0 --steps 20 >> gpurun_out/${TAG}_c3.log 2>&1
timeout 1500 python scripts/sweep_force.py --config c4 --libs variants/*.so --bins 0x0 --steps 8 >> gpurun_out/${TAG}_c4.log 2>&1
done
grep -h force_ms gpurun_out/${TAG}_*.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['lib'], d['n'], round(d['ms_per_step'],4), round(d['force_ms'],4))"
