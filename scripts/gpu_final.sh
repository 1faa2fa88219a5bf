#!/bin/bash
# Round-2 final check of the committed build: smoke, every GPU test, the default bench line,
# the C3 line, the launch list of one C2 fill and an ncu --set full capture of the sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
( time timeout 2400 python -m pytest tests -m gpu -x -q -rs ) > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-c4 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "rc=$?" >> gpurun_out/bench_c3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-clocks --no-c4"
timeout 300 $B > gpurun_out/plain_c2.json 2> gpurun_out/plain_c2.err && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_quad -s 20 -c 1 -o gpurun_out/prof_sweep_c2_final -f $B > gpurun_out/ncu_full_sweep.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full_sweep.log
