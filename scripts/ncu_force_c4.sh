mkdir -p gpurun_out
CMD="python bench.py --config c4 --n 16777216 --steps 2 --warmup 3 --no-cpu --no-e2e --bins 2"
$CMD > gpurun_out/ncu4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_force -s 3 -c 1 -o gpurun_out/prof_force_c4_flat -f $CMD > gpurun_out/ncu4_full.log 2>&1
tail -n 2 gpurun_out/ncu4_full.log; tail -c 600 gpurun_out/ncu4_plain.log
