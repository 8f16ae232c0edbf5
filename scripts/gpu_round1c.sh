mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r1e_pytest.log
timeout 900 python scripts/sweep_force.py --config c4 --bins 1x1 2x1 2x2 > gpurun_out/r1e_sweep_c4.log 2>&1
timeout 600 python scripts/sweep_force.py --config c1 --steps 50 --warmup 5 --bins 1x1 2x1 2x2 3x1 > gpurun_out/r1e_sweep_c1.log 2>&1
tail -n 20 gpurun_out/r1e_*.log
