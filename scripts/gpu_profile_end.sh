#!/bin/bash
# end-of-round profile evidence for the current build (c4 @ 2^26): launch list + one full k_force capture
mkdir -p gpurun_out
TAG=${TAG:-pe}
timeout 600 python bench.py --steps 3 --warmup 6 --no-cpu --no-e2e > gpurun_out/${TAG}_plain.json 2>&1 || { tail -3 gpurun_out/${TAG}_plain.json; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/${TAG}_launches_c4.csv \
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_force -s 8 -c 1 \
  -o gpurun_out/${TAG}_force_c4 -f python bench.py --steps 3 --warmup 6 --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_full.log 2>&1
ncu -i gpurun_out/${TAG}_force_c4.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_force_c4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_source.csv 2>/dev/null
python scripts/ncu_lines.py gpurun_out/${TAG}_source.csv 40 > gpurun_out/${TAG}_lines.txt
tail -1 gpurun_out/${TAG}_ncu_full.log; head -3 gpurun_out/${TAG}_lines.txt
