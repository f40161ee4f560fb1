cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python scripts/time_cfg.py 3 1 > gpurun_out/ncu_c3.log 2>&1
