cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 1 2 3 4 5; do timeout 300 python scripts/time_cfg.py $c 5 >> gpurun_out/time_cfg.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/time_cfg.py 5 1 > gpurun_out/ncu_c5.log 2>&1
