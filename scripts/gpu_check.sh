#!/bin/bash
# re-entry check: GPU parity suite, smoke, default bench line, short c1/c3/c5 lines
mkdir -p gpurun_out
TAG=${TAG:-chk}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
for c in c1 c3 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
tail -3 gpurun_out/${TAG}_pytest.log; tail -1 gpurun_out/${TAG}_smoke.log; cat gpurun_out/${TAG}_bench_*.json
