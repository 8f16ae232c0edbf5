#!/bin/bash
# c2 at its defined shape (200 iterations from 4,096 cells), decomposition overhead at N = 1 (c4 weak, c3)
mkdir -p gpurun_out
TAG=${TAG:-r2m}
timeout 1500 python bench.py --config c2 --steps 197 --warmup 3 > gpurun_out/${TAG}_bench_c2_full.json 2> gpurun_out/${TAG}_bench_c2_full.err
timeout 900 python bench.py --decompose --no-cpu --no-e2e > gpurun_out/${TAG}_bench_c4_dec.json 2> gpurun_out/${TAG}_bench_c4_dec.err
timeout 900 python bench.py --config c3 --decompose --no-cpu --no-e2e > gpurun_out/${TAG}_bench_c3_dec.json 2> gpurun_out/${TAG}_bench_c3_dec.err
timeout 900 python bench.py --config c3 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/${TAG}_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        e=d.get("e2e") or {}
        r=d.get("roofline") or {}
        print(f, "%.4g"%d["value"], "%.4f ms"%d["ms_per_step"], "e2e %.4g"%(e.get("value") or 0), "cpu", (d.get("cpu_baseline") or {}), "kernel", r.get("kernel"), "frac", r.get("frac"), d.get("config"))
    except Exception as ex: print(f, "ERR", ex); print(open(f.replace(".json",".err")).read()[-800:])
PY
