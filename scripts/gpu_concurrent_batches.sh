#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/concurrent_batches.py 8192 > gpurun_out/conc.json 2> gpurun_out/conc.err
MPR_SWEEP_WAVES=1 timeout 900 python scripts/concurrent_batches.py 8192 >> gpurun_out/conc.json 2>> gpurun_out/conc.err
