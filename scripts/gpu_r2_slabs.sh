#!/bin/bash
# Round 2: the in-library multi-rank paths (row slabs, realization shards) on the GPU.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "row_slabs or realization_shards or nccl or lifecycle or ordered_reduce or adaptive_realization" > gpurun_out/pytest_slabs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_slabs.log
timeout 300 python scripts/sanitize_case.py > gpurun_out/sanitize_case.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_case.log
