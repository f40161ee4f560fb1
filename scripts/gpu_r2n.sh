cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/n_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/n_pytest_gpu.log
for c in 1 2 3 4 5; do timeout 300 python scripts/time_cfg.py $c 5 >> gpurun_out/n_time.log 2>&1; done
