#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B="python bench.py --config C4 --steps 1 --warmup 1 --no-c4 --no-e2e --no-cpu-baseline --no-clocks"
timeout 600 $B > gpurun_out/c4_plain.json 2> gpurun_out/c4_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_smooth_wide|k_smooth_rs|k_block_stats4|k_init_states|k_acc_reduce|k_predict4" -c 8 -o gpurun_out/prof_params2_c4 -f $B > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
