cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 1 2; do timeout 300 python scripts/time_cfg.py $c 5 >> gpurun_out/time_cfg.log 2>&1; done
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c4 > gpurun_out/bench_small.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_interp_top_smem|k_fused_bottom|k_eval_top_rows" -c 3 -o gpurun_out/prof_c2_r2 python scripts/prof_c2.py 1 > gpurun_out/ncu_full.log 2>&1
