#!/bin/bash
# end-of-round evidence: GPU suite, smoke, default bench (c4 with CPU baseline), the other configs,
# the reference arm, the launch list of the default bench and one full k_force capture
mkdir -p gpurun_out
TAG=${TAG:-fin}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
for c in c1 c3 c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 900 python bench.py --config c2 --steps 20 --warmup 150 --no-cpu > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref_c4.json 2> gpurun_out/${TAG}_ref_c4.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/${TAG}_launches_c4.csv \
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_force -s 8 -c 1 \
  -o gpurun_out/${TAG}_force_c4 -f python bench.py --steps 3 --warmup 6 --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_full.log 2>&1
ncu -i gpurun_out/${TAG}_force_c4.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_force_c4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_source.csv 2>/dev/null
python scripts/ncu_lines.py gpurun_out/${TAG}_source.csv 40 > gpurun_out/${TAG}_lines.txt
python scripts/launch_summary.py gpurun_out/${TAG}_launches_c4.csv > gpurun_out/${TAG}_launch_summary.txt
tail -2 gpurun_out/${TAG}_pytest.log; tail -1 gpurun_out/${TAG}_smoke.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/fin_bench_*.json")) + ["gpurun_out/fin_ref_c4.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        e=d.get("e2e") or {}
        print(f, "%.4g"%d["value"], "%.4f"%d["ms_per_step"], "e2e %.4g"%(e.get("value") or 0), "cpu", (d.get("cpu_baseline") or {}).get("value"), "frac", (d.get("roofline") or {}).get("frac"))
    except Exception as ex: print(f, "ERR", ex)
PY
head -12 gpurun_out/${TAG}_launch_summary.txt
