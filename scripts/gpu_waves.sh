#!/bin/bash
# Resident-wave count for the default variant at C2 and C4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in 2 3 4 6; do
  MPR_SWEEP_WAVES=$w timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-c4 --no-e2e --no-clocks > gpurun_out/w2_c2_$w.json 2>/dev/null
done
for w in 8 16 32 64; do
  MPR_SWEEP_WAVES=$w timeout 600 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --no-e2e --no-clocks > gpurun_out/w2_c4_$w.json 2>/dev/null
done
