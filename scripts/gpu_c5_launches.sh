# C5 launch list (one product)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python scripts/time_cfg.py 5 1 > /dev/null 2>&1
