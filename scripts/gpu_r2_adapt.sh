#!/bin/bash
# Adaptive protocol timing (2048^2, p = 0.85, M = 100) with one-wave and multi-wave energy launches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/adaptive_timing.py 28 > gpurun_out/adapt_w1.jsonl 2> gpurun_out/adapt_w1.err
MPR_ENERGY_WAVES=1 timeout 600 python scripts/adaptive_timing.py 28 > gpurun_out/adapt_wN.jsonl 2> gpurun_out/adapt_wN.err
MPR_ENERGY_WAVES=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "adaptive or energy or c1_config" > gpurun_out/pytest_ew.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ew.log
