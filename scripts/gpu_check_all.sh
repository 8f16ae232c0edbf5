#!/bin/bash
# full GPU suite + smoke + c4/c1 bench lines (lists auto and off)
mkdir -p gpurun_out
TAG=${TAG:-chk}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_gpu.log
tail -3 gpurun_out/${TAG}_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for a in "--config c4" "--config c4 --lists off" "--config c1" "--config c1 --lists off"; do
  timeout 600 python bench.py $a --no-cpu --no-e2e 2>/dev/null | tail -1 > gpurun_out/${TAG}_tmp.json
  python -c "
import json
d=json.loads(open('gpurun_out/${TAG}_tmp.json').read())
print('$a', '%.4g agent-it/s %.4f ms/step force %.3f ms' % (d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms']), d.get('lists'))
"
done
