cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 4 5; do timeout 200 python scripts/time_cfg.py $c 3 >> gpurun_out/time_cfg.log 2>&1; done
