cd $GRAFT_REPO_ROOT
NCU=1 STEPS=20 bash scripts/gpu_check.sh
KERNEL="k_sweep_quad" TAG=final2 SKIP=20 COUNT=2 bash scripts/gpu_ncu_full.sh
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san_$tool.log
done
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
