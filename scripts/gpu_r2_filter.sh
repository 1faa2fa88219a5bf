#!/bin/bash
# Round 2: the SFU-filtered sweep kernel (variant 40): its tests, the whole GPU suite, and
# the bench with the filter (default) and without it (variant 28).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "filter or every_sweep_variant" > gpurun_out/pytest_filter.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_filter.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench40.json 2> gpurun_out/bench40.err; echo "rc=$?" >> gpurun_out/bench40.err
MPR_SWEEP_VARIANT=28 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench28.json 2> gpurun_out/bench28.err; echo "rc=$?" >> gpurun_out/bench28.err
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
