#!/bin/bash
# A/B of the current build: sweep-kernel tests first, then C2 and C4 bench lines (VARIANTS).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "every_sweep_variant or split_tail or multiwave or adaptive or c1_config or energy or n_avg or fuzz_small" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
for v in ${VARIANTS:-28}; do
  MPR_SWEEP_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --no-e2e > gpurun_out/ab_c2_v$v.json 2> gpurun_out/ab_c2_v$v.err
  MPR_SWEEP_VARIANT=$v timeout 600 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --no-e2e > gpurun_out/ab_c4_v$v.json 2> gpurun_out/ab_c4_v$v.err
done
