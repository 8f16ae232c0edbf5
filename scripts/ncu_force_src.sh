#!/bin/bash
# full ncu capture of k_force at c4 2^24 with source correlation, exported as CSV
mkdir -p gpurun_out
TAG=${TAG:-src}
CMD="python bench.py --config c4 --n 16777216 --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { tail -5 gpurun_out/${TAG}_plain.log; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_force -s 3 -c 1 -o gpurun_out/${TAG}_force -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_force.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_force.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
python scripts/ncu_lines.py gpurun_out/${TAG}_source.csv 60 > gpurun_out/${TAG}_lines.txt
head -40 gpurun_out/${TAG}_lines.txt
