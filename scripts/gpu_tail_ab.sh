#!/bin/bash
# The odd-pair fallback (C4 tail batch; M = 4k + 2 on small grids): variant 13 vs 14.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "every_sweep_variant or split_tail or multiwave or c1_config or ragged or fuzz_small" > gpurun_out/pytest_tail.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tail.log
for i in 1 2; do
  for t in 13 14; do
    MPR_TAIL_VARIANT=$t timeout 600 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --no-e2e --no-clocks > gpurun_out/tail_c4_t${t}_$i.json 2>/dev/null
    MPR_TAIL_VARIANT=$t timeout 300 python bench.py --M 10 --steps 20 --warmup 3 --no-cpu-baseline --no-c4 --no-e2e --no-clocks > gpurun_out/tail_c2m10_t${t}_$i.json 2>/dev/null
  done
done
