mkdir -p gpurun_out
TAG=${TAG:-v}
for L in variants/*.so; do ABSIM_GPU_LIB=$PWD/$L timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x 2>&1 | tail -1 | sed "s#^#$L #" >> gpurun_out/${TAG}_pytest.log; done
timeout 1200 python scripts/sweep_force.py --config c4 --n 16777216 --libs variants/*.so --bins 2x2 > gpurun_out/${TAG}_sweep_c4.log 2>&1
timeout 600 python scripts/sweep_force.py --config c1 --steps 50 --warmup 5 --libs variants/*.so --bins 1x1 2x2 > gpurun_out/${TAG}_sweep_c1.log 2>&1
tail -n 12 gpurun_out/${TAG}_*.log
