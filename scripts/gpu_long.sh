cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "long or c5 or c4" > gpurun_out/pytest_long.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_long.log
timeout 300 python scripts/time_cfg.py 4 3 > gpurun_out/time_cfg.log 2>&1
