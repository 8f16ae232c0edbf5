# round evidence: tests, smoke, bench lines for every config, reference arm, ncu
mkdir -p gpurun_out
T=${TAG:-ev}
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_ref_c4.json 2> gpurun_out/${T}_ref_c4.err
timeout 600 python bench.py --config c1 --steps 100 --warmup 5 > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err
timeout 900 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 900 python bench.py --config c5 --steps 30 --warmup 3 > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
timeout 900 python bench.py --config c2 --steps 200 --warmup 0 --no-e2e > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/${T}_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_launches_c4.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
$CMD > gpurun_out/${T}_ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_force -s 3 -c 1 -o gpurun_out/${T}_force_c4 -f $CMD > gpurun_out/${T}_ncu_full.log 2>&1
cat gpurun_out/${T}_pytest.log gpurun_out/${T}_smoke.log
