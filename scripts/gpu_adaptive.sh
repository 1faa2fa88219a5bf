#!/bin/bash
# Adaptive protocol timing (2048^2, p = 0.85, M = 100) on the current build.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/adaptive_timing.py ${VARIANTS:-33} > gpurun_out/adaptive_timing.jsonl 2> gpurun_out/adaptive_timing.err
