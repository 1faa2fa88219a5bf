#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "split_tail or every_sweep_variant or fuzz_small or c1_config or c4_full or row_slabs_distributed or adaptive" > gpurun_out/pytest_tail.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tail.log
B="python bench.py --config C4 --steps 3 --warmup 2 --no-c4 --no-cpu-baseline"
timeout 600 $B > gpurun_out/c4_tail.json 2> gpurun_out/c4_tail.err
B="python bench.py --config C4 --steps 1 --warmup 1 --no-c4 --no-e2e --no-cpu-baseline --no-clocks"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c4.log
