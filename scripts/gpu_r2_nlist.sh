#!/bin/bash
# round 2: neighbour-list path — parity, then c4 / c1 with and without lists
mkdir -p gpurun_out
TAG=${TAG:-r2a}
timeout 600 python -m pytest tests/test_nlist.py -x -q > gpurun_out/${TAG}_nlist.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_nlist.log
tail -3 gpurun_out/${TAG}_nlist.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_gpu.log
tail -3 gpurun_out/${TAG}_gpu.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err
ABSIM_NLIST=0 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/${TAG}_c4_nolist.json 2> gpurun_out/${TAG}_c4_nolist.err
timeout 600 python bench.py --config c1 --no-cpu --no-e2e > gpurun_out/${TAG}_c1.json 2> gpurun_out/${TAG}_c1.err
ABSIM_NLIST=0 timeout 600 python bench.py --config c1 --no-cpu --no-e2e > gpurun_out/${TAG}_c1_nolist.json 2> gpurun_out/${TAG}_c1_nolist.err
for f in gpurun_out/${TAG}_c*.json; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('%.4g agent-it/s  %.3f ms/step  force %.3f ms frac %.4f' % (d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac']), d.get('lists'))
" 2>&1 | tail -2; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_c4.csv \
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/${TAG}_launches_c4.csv > gpurun_out/${TAG}_launch_summary.txt 2>&1
head -20 gpurun_out/${TAG}_launch_summary.txt
