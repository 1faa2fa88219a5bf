#!/bin/bash
# Randomised parity campaign on the final build (the fuzz tests scaled up).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( time MPR_FUZZ_CASES=3000 MPR_FUZZ_ADAPTIVE_CASES=300 MPR_FUZZ_SLAB_CASES=100 timeout 3000 python -m pytest tests/test_gpu_parity.py -q -k "fuzz" ) > gpurun_out/fuzz.log 2>&1; echo "rc=$?" >> gpurun_out/fuzz.log
( time MPR_SWEEP_WAVES=6 MPR_FUZZ_CASES=1000 timeout 1800 python -m pytest tests/test_gpu_parity.py -q -k "fuzz_small" ) > gpurun_out/fuzz_waves.log 2>&1; echo "rc=$?" >> gpurun_out/fuzz_waves.log
