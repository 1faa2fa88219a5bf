#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "mixed or split_tail or every_sweep or c1_config or ragged" > gpurun_out/pytest_mix.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mix.log
timeout 600 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --no-e2e > gpurun_out/ab_c4_mix.json 2> gpurun_out/ab_c4_mix.err
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --no-e2e --M 10 > gpurun_out/ab_c2m10_mix.json 2> gpurun_out/ab_c2m10_mix.err
MPR_SPLIT_MIN_P=0 MPR_SWEEP_VARIANT=28 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --no-e2e --M 10 > gpurun_out/ab_c2m10_ref.json 2> gpurun_out/ab_c2m10_ref.err
