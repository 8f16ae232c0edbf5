#!/bin/bash
# quick loop: list tests, c4 and c1 bench lines, c4 launch list
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 600 python -m pytest tests/test_nlist.py -x -q > gpurun_out/${TAG}_nlist.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_nlist.log
tail -3 gpurun_out/${TAG}_nlist.log
for c in c4 c1; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err
  python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_$c.json').read().strip().splitlines()[-1])
print('$c %.4g agent-it/s  %.3f ms/step  force %.3f ms frac %.4f' % (d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac']), d.get('lists'))
" 2>&1 | tail -1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_c4.csv \
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/${TAG}_launches_c4.csv > gpurun_out/${TAG}_launch_summary.txt 2>&1
head -8 gpurun_out/${TAG}_launch_summary.txt
