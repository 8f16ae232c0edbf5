# one ncu --set full capture of the force kernel (c1, 131k agents) + launch list
mkdir -p gpurun_out
CMD="python bench.py --config c1 --steps 5 --warmup 3 --no-cpu --no-e2e --bins 0"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_force -s 3 -c 1 -o gpurun_out/prof_force_c1_box -f $CMD > gpurun_out/ncu_full.log 2>&1
$CMD > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c1_box.csv $CMD > gpurun_out/ncu_launch.log 2>&1
tail -n 3 gpurun_out/ncu_full.log
