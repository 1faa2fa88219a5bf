cd $GRAFT_REPO_ROOT
NCU=1 STEPS=20 bash scripts/gpu_check.sh
KERNEL="k_sweep_quad" TAG=final2 SKIP=20 COUNT=2 bash scripts/gpu_ncu_full.sh
# compute-sanitizer is closed on the GPU pool; scripts/sanitize_case.py is kept for local use
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in C3 C4; do timeout 400 python scripts/sweep_variants.py --config $c --variants 28,13 --rounds 1 > gpurun_out/sv_final_$c.log 2>&1; done
