#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-sk}
run() { timeout 600 python bench.py --no-cpu --no-e2e "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$*', '%.3f ms/step' % d['ms_per_step'], 'force %.2f' % d['roofline']['avg_launch_ms'], d.get('lists'))
"; }
run --lists off
run --skin 2.7
run --skin 4
run --skin 5.5
run --lists off --warmup 28
run --skin 2.7 --warmup 28
run --skin 4 --warmup 28
run --config c1 --lists off
run --config c1 --skin 1.8
run --config c1 --skin 3
run --config c1 --lists off --warmup 50
run --config c1 --skin 1.8 --warmup 50
