#!/bin/bash
# Repeated A/B of two sweep variants at C2 and C4 (alternating runs).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in ${VARIANTS:-28 33}; do
    MPR_SWEEP_VARIANT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-c4 --no-e2e --no-clocks > gpurun_out/rep_c2_v${v}_$i.json 2>/dev/null
  done
done
for i in 1 2; do
  for v in ${VARIANTS:-28 33}; do
    MPR_SWEEP_VARIANT=$v timeout 600 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --no-e2e --no-clocks > gpurun_out/rep_c4_v${v}_$i.json 2>/dev/null
  done
done
