cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/time_cfg.py 5 1 > gpurun_out/plain_c5.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/time_cfg.py 5 1 > gpurun_out/ncu_c5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/ncu_c4.log 2>&1
