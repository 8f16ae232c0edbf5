#!/bin/bash
# round-2 evidence: GPU suite, smoke, default bench (c4 with CPU baseline + e2e), the reference arm, lists off,
# other configs, launch list of the default bench, full ncu capture of the list kernels and the walk
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
timeout 900 python bench.py --lists off --no-cpu --no-e2e > gpurun_out/${TAG}_bench_c4_nolist.json 2> gpurun_out/${TAG}_bench_c4_nolist.err
timeout 900 python bench.py --steps 47 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_c4_50steps.json 2> gpurun_out/${TAG}_bench_c4_50steps.err
for c in c1 c3 c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref_c4.json 2> gpurun_out/${TAG}_ref_c4.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/${TAG}_launches_c4.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/${TAG}_launches_c4.csv > gpurun_out/${TAG}_launch_summary.txt
tail -2 gpurun_out/${TAG}_pytest.log; tail -1 gpurun_out/${TAG}_smoke.log
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/${TAG}_bench_*.json"))+["gpurun_out/${TAG}_ref_c4.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        e=d.get("e2e") or {}
        r=d.get("roofline") or {}
        print(f, "%.4g"%d["value"], "%.4f ms"%d["ms_per_step"], "e2e %.4g"%(e.get("value") or 0), "cpu", (d.get("cpu_baseline") or {}).get("value"), "kernel", r.get("kernel"), "frac", r.get("frac"), d.get("lists"))
    except Exception as ex: print(f, "ERR", ex)
PY
head -16 gpurun_out/${TAG}_launch_summary.txt
KERNELS="k_list_build k_list_scan k_list_forces k_force" TAG=${TAG}n bash scripts/ncu_r2_lists.sh
