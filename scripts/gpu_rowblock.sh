#!/bin/bash
# blocked bin-row order: parity suite, then k_force / step time vs ABSIM_ROW_BLOCK
mkdir -p gpurun_out
TAG=${TAG:-rb}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
for RB in 0 8 16 32 64; do
  ABSIM_ROW_BLOCK=$RB timeout 900 python scripts/sweep_force.py --config c4 --bins 0x0 --steps 5 | sed "s/^/rb=$RB /" >> gpurun_out/${TAG}_c4_26.log 2>&1
done
for RB in 0 16; do
  ABSIM_ROW_BLOCK=$RB timeout 900 python scripts/sweep_force.py --config c4 --n 16777216 --bins 0x0 | sed "s/^/rb=$RB /" >> gpurun_out/${TAG}_c4_24.log 2>&1
  ABSIM_ROW_BLOCK=$RB timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu --no-e2e | sed "s/^/rb=$RB /" >> gpurun_out/${TAG}_c5.log 2>&1
  ABSIM_ROW_BLOCK=$RB timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --no-e2e | sed "s/^/rb=$RB /" >> gpurun_out/${TAG}_c3.log 2>&1
done
grep -h "force_ms\|\"value\"" gpurun_out/${TAG}_c*.log | cut -c1-260
