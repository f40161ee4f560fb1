cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 1 2 3 4; do timeout 120 python scripts/time_cfg.py $c 5 >> gpurun_out/time_cfg.log 2>&1; done
timeout 300 ncu --set full --clock-control none --import-source on -k "regex:k_fused_bottom" -c 1 -o gpurun_out/prof_fused3 python scripts/prof_c2.py 1 > gpurun_out/ncu_full_c2.log 2>&1
