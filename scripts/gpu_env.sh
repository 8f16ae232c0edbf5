#!/bin/bash
# environments: GPU parity suite (incl. brute-force env), then grid vs brute-force at c1
mkdir -p gpurun_out
TAG=${TAG:-env}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --config c1 --steps 20 --warmup 3 > gpurun_out/${TAG}_c1_grid.json 2> gpurun_out/${TAG}_c1_grid.err
timeout 900 python bench.py --config c1 --steps 5 --warmup 3 --env brute_force > gpurun_out/${TAG}_c1_brute.json 2> gpurun_out/${TAG}_c1_brute.err
timeout 900 python bench.py --config c1 --impl reference --steps 3 --warmup 1 --env brute_force > gpurun_out/${TAG}_c1_brute_ref.json 2> gpurun_out/${TAG}_c1_brute_ref.err
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/env_c1_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d.get("cpu_baseline",{}).get("value"), d.get("roofline",{}).get("avg_launch_ms"))
    except Exception as e: print(f, "ERR", e)
PY
tail -3 gpurun_out/${TAG}_c1_brute.err
