cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf -x -k "t16 or B-16 or 16- or c5 or stage or sharded" > gpurun_out/i_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/i_pytest_gpu.log
timeout 300 python scripts/time_cfg.py 5 3 >> gpurun_out/i_time.log 2>&1
TOOM_T16_MATRIX=0 timeout 300 python scripts/time_cfg.py 5 3 >> gpurun_out/i_time.log 2>&1
