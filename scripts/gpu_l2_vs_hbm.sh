#!/bin/bash
# Is the sweep limited by HBM? The C2 grid with the state L2-resident (M = 24: 33 MB) vs
# streamed from HBM (M = 100: 138 MB; M = 400: 553 MB): per-update sweep rates.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for M in 24 48 100 200 400; do
  timeout 300 python bench.py --M $M --steps 5 --warmup 3 --no-cpu-baseline --no-c4 --no-e2e > gpurun_out/l2_m$M.json 2> gpurun_out/l2_m$M.err
done
