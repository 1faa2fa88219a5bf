#!/bin/bash
# A/B of sweep variants at C2 and C4 (VARIANTS), bench lines per variant; variant tests first.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_sweep_variant or split_tail" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
for v in ${VARIANTS:-28 30}; do
  MPR_SWEEP_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --no-e2e > gpurun_out/ab_c2_v$v.json 2> gpurun_out/ab_c2_v$v.err
  MPR_SWEEP_VARIANT=$v timeout 600 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --no-e2e > gpurun_out/ab_c4_v$v.json 2> gpurun_out/ab_c4_v$v.err
done
