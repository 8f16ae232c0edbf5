#!/bin/bash
# quick parity + step times of every config (no CPU baseline, no e2e)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_nlist.py tests/test_golden.py tests/test_reference_models.py tests/test_sir.py tests/test_environments.py -m gpu -q -x 2>&1 | tail -2
for a in "--config c4 --lists off" "--config c4" "--config c1 --steps 95 --warmup 5" "--config c1 --steps 95 --warmup 5 --lists off" "--config c3" "--config c5" "--config c2 --steps 197 --warmup 3"; do
  timeout 900 python bench.py $a --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$a: %.4g agent-it/s %.4f ms/step kernel %.4f ms'%(d['value'],d['ms_per_step'],d['roofline']['avg_launch_ms']), d['lists']['builds'], d['lists']['list_steps'])"
done
