set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1
timeout 600 python bench.py --config c1 --steps 50 --warmup 5 --bins 1 --no-cpu > gpurun_out/r1_bench_c1_b1.log 2>&1
timeout 600 python bench.py --config c1 --steps 50 --warmup 5 --bins 2 --no-cpu --no-e2e > gpurun_out/r1_bench_c1_b2.log 2>&1
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --bins 1 --no-cpu --no-e2e > gpurun_out/r1_bench_c4_b1.log 2>&1
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --bins 2 --no-cpu --no-e2e > gpurun_out/r1_bench_c4_b2.log 2>&1
tail -n 40 gpurun_out/r1_*.log
