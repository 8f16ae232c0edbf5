#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-r2c2}
CMD="python bench.py --config c2 --steps 197 --warmup 3 --no-cpu --no-e2e"
k=k_force
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^$k -s ${SKIP:-196} -c 1 -o /tmp/${TAG}_$k -f $CMD > gpurun_out/${TAG}_ncu_$k.log 2>&1
ncu -i /tmp/${TAG}_$k.ncu-rep --page details > gpurun_out/${TAG}_${k}_details.txt 2>/dev/null
ncu -i /tmp/${TAG}_$k.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${TAG}_${k}_source.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/${TAG}_${k}_source.csv 30 > gpurun_out/${TAG}_${k}_lines.txt 2>&1
grep -E "Duration|Registers Per|Achieved Occupancy|Executed Ipc Active|Issue Slots Busy|Grid Size|Block Size|Waves Per SM|Theoretical Occ|SM Active Cycles|Elapsed Cycles|Avg. Active Threads|k_force" gpurun_out/${TAG}_${k}_details.txt | head -14
head -32 gpurun_out/${TAG}_${k}_lines.txt
rm -f /tmp/${TAG}_$k.ncu-rep /tmp/${TAG}_${k}_source.csv
