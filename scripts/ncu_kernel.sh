#!/bin/bash
# full ncu capture of one kernel of one config: scripts/ncu_kernel.sh <config> <kernel> [skip]
mkdir -p gpurun_out
CFG=$1; K=$2; SKIP=${3:-10}; TAG=${TAG:-r2k}
CMD="python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^$K -s $SKIP -c 1 -o /tmp/${TAG}_$K -f $CMD > gpurun_out/${TAG}_ncu_$K.log 2>&1
ncu -i /tmp/${TAG}_$K.ncu-rep --page details > gpurun_out/${TAG}_${CFG}_${K}_details.txt 2>/dev/null
ncu -i /tmp/${TAG}_$K.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${TAG}_${K}_source.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/${TAG}_${K}_source.csv 30 > gpurun_out/${TAG}_${CFG}_${K}_lines.txt 2>&1
grep -E "Duration|Registers Per|Achieved Occupancy|Executed Ipc Active|Issue Slots Busy|Avg. Active Threads|DRAM Throughput|L1/TEX Hit|L2 Hit" gpurun_out/${TAG}_${CFG}_${K}_details.txt | head -10
head -28 gpurun_out/${TAG}_${CFG}_${K}_lines.txt
rm -f /tmp/${TAG}_$K.ncu-rep /tmp/${TAG}_${K}_source.csv
