#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-r2c1}
CMD="python bench.py --config c1 --steps 40 --warmup 5 --no-cpu --no-e2e"
for k in ${KERNELS:-k_list_forces k_reduce_finalize k_list_scan}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:^$k -s 30 -c 1 -o /tmp/${TAG}_$k -f $CMD > gpurun_out/${TAG}_ncu_$k.log 2>&1
  ncu -i /tmp/${TAG}_$k.ncu-rep --page details > gpurun_out/${TAG}_${k}_details.txt 2>/dev/null
  ncu -i /tmp/${TAG}_$k.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${TAG}_${k}_source.csv 2>/dev/null
  python scripts/ncu_lines.py /tmp/${TAG}_${k}_source.csv 25 > gpurun_out/${TAG}_${k}_lines.txt 2>&1
  echo "== $k"; grep -E "Duration|Registers Per|Achieved Occupancy|Executed Ipc Active|Issue Slots Busy|Grid Size|Block Size|Waves Per SM|Theoretical Occ" gpurun_out/${TAG}_${k}_details.txt | head -12
  head -14 gpurun_out/${TAG}_${k}_lines.txt
  rm -f /tmp/${TAG}_$k.ncu-rep /tmp/${TAG}_${k}_source.csv
done
