#!/bin/bash
# round-2 evidence: bench lines for every config + one full ncu capture of k_force at c4
for c in c1 c3 c5 c2; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2b_$c.json 2> gpurun_out/r2b_$c.err || tail -3 gpurun_out/r2b_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_force -s 8 -c 1 \
  -o gpurun_out/r2b_force_c4 python bench.py --steps 3 --warmup 6 --no-cpu --no-e2e > gpurun_out/r2b_ncu.log 2>&1
tail -2 gpurun_out/r2b_ncu.log
