mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r1b_pytest.log
timeout 1500 python scripts/sweep_force.py --config c4 --libs variants/*.so --bins 1x1 2x1 3x1 2x2 > gpurun_out/r1b_sweep_c4.log 2>&1
timeout 600 python scripts/sweep_force.py --config c1 --steps 50 --warmup 5 --libs variants/*.so --bins 1x1 2x1 2x2 > gpurun_out/r1b_sweep_c1.log 2>&1
tail -n 40 gpurun_out/r1b_*.log
