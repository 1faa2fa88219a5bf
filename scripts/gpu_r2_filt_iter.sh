#!/bin/bash
# Iteration on the filtered sweep kernel: its tests, a C2 bench per variant, one ncu capture.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "filter or every_sweep_variant" > gpurun_out/pytest_filter.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_filter.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --no-e2e"
for v in ${VARIANTS:-28 40 42 43 44}; do
  MPR_SWEEP_VARIANT=$v timeout 300 $B > gpurun_out/bench$v.json 2> gpurun_out/bench$v.err; echo "rc=$?" >> gpurun_out/bench$v.err
done
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-clocks --no-c4"
MPR_SWEEP_VARIANT=${NCU_VARIANT:-43} timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-k_sweep_filt} -s 10 -c 1 \
  -o gpurun_out/prof_filt_c2 -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
