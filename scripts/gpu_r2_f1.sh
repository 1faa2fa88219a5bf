#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "adaptive or row_slabs_distributed" > gpurun_out/pytest_f1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f1.log
timeout 1500 python scripts/f1_equilibrium.py > gpurun_out/f1_equilibrium.jsonl 2> gpurun_out/f1_equilibrium.err; echo "rc=$?" >> gpurun_out/f1_equilibrium.err
