#!/bin/bash
# full GPU suite (no -x) + list policy sweep on c4 (min steps x skin)
mkdir -p gpurun_out
TAG=${TAG:-r2b}
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -5 gpurun_out/${TAG}_pytest.log
for ms in 1.5 2 3; do for skin in 2 3 4.5; do
  ABSIM_LIST_MIN_STEPS=$ms timeout 600 python bench.py --no-cpu --no-e2e --skin $skin 2>/dev/null | tail -1 > gpurun_out/${TAG}_sw_${ms}_${skin}.json
  python - <<PY
import json
d=json.loads(open("gpurun_out/${TAG}_sw_${ms}_${skin}.json").read())
print("min_steps $ms skin $skin: %.4g agent-it/s %.3f ms/step list-step %.3f ms"%(d["value"],d["ms_per_step"],d["roofline"]["avg_launch_ms"]), d.get("lists"))
PY
done; done
