#!/bin/bash
# Grid-size experiment for the half-sweep kernel: resident waves of CTAs per launch.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in 4 8 16 32; do
  MPR_SWEEP_WAVES=$w timeout 600 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --no-e2e > gpurun_out/bench_c4_w$w.json 2> gpurun_out/bench_c4_w$w.err
done
for w in 1 2 4 8 16; do
  MPR_SWEEP_WAVES=$w timeout 600 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-c4 --no-e2e > gpurun_out/bench_c3_w$w.json 2> gpurun_out/bench_c3_w$w.err
done
