#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-r2c1}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --config c1 --steps 40 --warmup 5 --no-cpu --no-e2e $EXTRA > gpurun_out/${TAG}_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/${TAG}_launches.csv 200 > gpurun_out/${TAG}_summary.txt; cat gpurun_out/${TAG}_summary.txt
for i in 1 2 3; do python bench.py --config c1 --steps 100 --warmup 5 --no-cpu --no-e2e $EXTRA 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('%.4g agent-it/s %.4f ms/step'%(d['value'],d['ms_per_step']), d['lists'])"; done
