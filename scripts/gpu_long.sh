cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "long or stage or signed or sharded or c5 or c4" > gpurun_out/pytest_long.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_long.log
for c in 4 5; do timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/time_cfg.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/time_cfg.py 5 1 > gpurun_out/ncu_c5.log 2>&1
