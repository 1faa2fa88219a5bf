#!/bin/bash
# ncu --set full capture of the hot kernel (after the same command exits 0 without ncu).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-clocks ${BENCH_ARGS}"
timeout 300 $CMD > gpurun_out/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_sweep_half} -s ${SKIP:-10} -c ${COUNT:-2} \
  -o gpurun_out/prof_${TAG:-sweep} -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
