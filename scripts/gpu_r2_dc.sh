#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "dc or fuzz_small" > gpurun_out/pytest_dc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dc.log
timeout 600 python scripts/micro/order_timing.py > gpurun_out/order_timing.log 2>&1; echo "rc=$?" >> gpurun_out/order_timing.log
