cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/ncu_c4.log 2>&1
timeout 300 python scripts/sanitize_small.py > gpurun_out/sanitize_small.log 2>&1
