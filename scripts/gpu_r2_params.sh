#!/bin/bash
# Round 2: parity of the rewritten parameter-stage kernels, then the C4 launch list (one fill).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B="python bench.py --config C4 --steps 1 --warmup 1 --no-c4 --no-e2e --no-cpu-baseline --no-clocks"
timeout 600 $B > gpurun_out/c4_plain.json 2> gpurun_out/c4_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c4.log
