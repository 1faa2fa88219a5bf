#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --no-e2e --M 10"
timeout 300 $B > gpurun_out/ab_c2m10_mix.json 2> gpurun_out/ab_c2m10_mix.err
MPR_NO_MIX=1 MPR_SPLIT_MIN_P=0 timeout 300 $B > gpurun_out/ab_c2m10_split.json 2> gpurun_out/ab_c2m10_split.err
MPR_NO_MIX=1 timeout 600 python bench.py --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --no-e2e > gpurun_out/ab_c4_split.json 2> gpurun_out/ab_c4_split.err
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-clocks --no-c4 --M 10"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_mix -s 10 -c 1 -o gpurun_out/prof_mix -f $CMD > gpurun_out/ncu_mix.log 2>&1
MPR_NO_MIX=1 MPR_SPLIT_MIN_P=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 20 -c 2 -o gpurun_out/prof_split -f $CMD > gpurun_out/ncu_split.log 2>&1
