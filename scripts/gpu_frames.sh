#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-fr}
timeout 600 python -m pytest tests/test_frames.py -q -x > gpurun_out/${TAG}_frames.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_frames.log
tail -5 gpurun_out/${TAG}_frames.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --no-cpu > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
timeout 600 python bench.py --config c1 --steps 20 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_c1.json 2> gpurun_out/${TAG}_bench_c1.err
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/fr_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], json.dumps(d["e2e"])[:600])
    except Exception as e: print(f, "ERR", e)
PY
tail -5 gpurun_out/${TAG}_bench_c4.err
