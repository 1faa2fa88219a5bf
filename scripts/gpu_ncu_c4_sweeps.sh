#!/bin/bash
# ncu --set full of the C4 tail batch's one-pair half-sweep (k_sweep_half) and of the
# 8-realization batch's k_sweep_quad, one launch each (after the plain command exits 0).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-clocks --no-c4"
timeout 600 $B > gpurun_out/plain_c4.json 2> gpurun_out/plain_c4.err && \
timeout 1200 ncu --set full --clock-control none -k regex:"k_sweep_half|k_sweep_quad" -s 60 -c 2 -o gpurun_out/prof_c4_sweeps -f $B > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c4.log
