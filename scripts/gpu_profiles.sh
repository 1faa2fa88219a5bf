#!/bin/bash
# Round-2 profiles of the current build: launch lists of one C2 and one C4 fill, and an
# ncu --set full capture of the half-sweep kernel at C2 (each after the plain command exits 0).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-clocks --no-c4"
timeout 300 $B > gpurun_out/plain_c2.json 2> gpurun_out/plain_c2.err && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_quad -s 20 -c 1 -o gpurun_out/prof_sweep_c2_r02 -f $B > gpurun_out/ncu_full_sweep.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full_sweep.log
B4="python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-clocks --no-c4"
timeout 600 $B4 > gpurun_out/plain_c4.json 2> gpurun_out/plain_c4.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c4.csv $B4 > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c4.log
