mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/${TAG}_pytest.log
timeout 900 python scripts/sweep_force.py --config c4 --n 16777216 --bins 2x2 2x1 1x1 > gpurun_out/${TAG}_sweep_c4.log 2>&1
ABSIM_FORCE_KERNEL=tile timeout 900 python scripts/sweep_force.py --config c4 --n 16777216 --bins 2x2 >> gpurun_out/${TAG}_sweep_c4.log 2>&1
timeout 600 python scripts/sweep_force.py --config c1 --steps 50 --warmup 5 --bins 1x1 2x2 > gpurun_out/${TAG}_sweep_c1.log 2>&1
tail -n 12 gpurun_out/${TAG}_*.log
