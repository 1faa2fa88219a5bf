#!/bin/bash
# Round 2 full check: smoke, every GPU test (slow included), bench (C2 + C4 rows), the
# emulated 4-rank C4 line, the launch list of the bench command, a sweep ncu capture, and a
# compute-sanitizer attempt.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
free -g > gpurun_out/host_mem.txt 2>&1; nproc >> gpurun_out/host_mem.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --emulate 4 --config C4 --steps 2 --warmup 1 > gpurun_out/bench_emulate4.json 2> gpurun_out/bench_emulate4.err; echo "rc=$?" >> gpurun_out/bench_emulate4.err
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-clocks --no-c4"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_quad -s 20 -c 1 -o gpurun_out/prof_sweep_c2_r02 -f $B > gpurun_out/ncu_full_sweep.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full_sweep.log
timeout 600 compute-sanitizer --tool memcheck python scripts/sanitize_case.py > gpurun_out/sanitizer_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_memcheck.log
