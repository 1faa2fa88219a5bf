#!/bin/bash
# Adaptive protocol timing (2048^2, p = 0.85, M = 100): energy sweeps on variant 28 vs 33.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/adaptive_timing.py 33 > gpurun_out/adapt_e28.jsonl 2> gpurun_out/adapt_e28.err
MPR_ENERGY_33=1 timeout 600 python scripts/adaptive_timing.py 33 > gpurun_out/adapt_e33.jsonl 2> gpurun_out/adapt_e33.err
MPR_ENERGY_33=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "adaptive or energy or c1_config" > gpurun_out/pytest_e33.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_e33.log
