#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( time timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multiwave or every_sweep or split_tail or c1_config" ) > gpurun_out/pytest_mw.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mw.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --no-e2e > gpurun_out/mw_c2.json 2> gpurun_out/mw_c2.err
