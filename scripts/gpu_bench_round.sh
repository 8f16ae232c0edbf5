# round-end style run: tests, bench (default + c1), reference arm, ncu launch list + one full capture
mkdir -p gpurun_out
TAG=${TAG:-r1i}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
timeout 600 python bench.py --config c1 --steps 100 --warmup 5 --bins 1 --bins-x 1 > gpurun_out/${TAG}_bench_c1.json 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/${TAG}_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches_c4.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
$CMD > gpurun_out/${TAG}_ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_force -s 3 -c 1 -o gpurun_out/${TAG}_force_c4 -f $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
tail -n 5 gpurun_out/${TAG}_pytest.log gpurun_out/${TAG}_smoke.log; cat gpurun_out/${TAG}_bench.json gpurun_out/${TAG}_ref.json gpurun_out/${TAG}_bench_c1.json; tail -n 3 gpurun_out/${TAG}_bench.err gpurun_out/${TAG}_ref.err
