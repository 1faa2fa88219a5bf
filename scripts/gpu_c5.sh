#!/bin/bash
# BASELINE config 5 sweep on the current build (device and warm e2e from pinned buffers).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python scripts/sweep_c5.py --reps 3 > gpurun_out/c5_sweep.jsonl 2> gpurun_out/c5_sweep.err; echo "rc=$?" >> gpurun_out/c5_sweep.err
