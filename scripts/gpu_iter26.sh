cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 240 -k "p8 or c3 or ragged" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python scripts/time_cfg.py 3 1 > gpurun_out/ncu_c3.log 2>&1
timeout 200 python scripts/time_cfg.py 3 5 > gpurun_out/time_cfg.log 2>&1
