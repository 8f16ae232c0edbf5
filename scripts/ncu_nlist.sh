#!/bin/bash
# full ncu capture of the list force kernel (c4 @ 2^26)
mkdir -p gpurun_out
TAG=${TAG:-r2c}
CMD="python bench.py --steps 12 --warmup 3 --no-cpu --no-e2e"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_force_list -s 10 -c 1 -o gpurun_out/${TAG}_flist -f $CMD > gpurun_out/${TAG}_ncu1.log 2>&1
ncu -i gpurun_out/${TAG}_flist.ncu-rep --page details > gpurun_out/${TAG}_flist_details.txt 2>/dev/null
ncu -i gpurun_out/${TAG}_flist.ncu-rep --page raw --csv > gpurun_out/${TAG}_flist_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_flist.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_flist_source.csv 2>/dev/null
tail -n 3 gpurun_out/${TAG}_ncu1.log
