mkdir -p gpurun_out
TAG=${TAG:-r1f}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${TAG}_pytest.log
timeout 1500 python scripts/sweep_force.py --config c4 --n 16777216 --libs variants/*.so --bins 1x1 2x2 > gpurun_out/${TAG}_sweep_c4.log 2>&1
timeout 600 python scripts/sweep_force.py --config c1 --steps 50 --warmup 5 --libs variants/*.so --bins 1x1 2x2 > gpurun_out/${TAG}_sweep_c1.log 2>&1
tail -n 20 gpurun_out/${TAG}_*.log
