# C3 launch list (time, DRAM bytes, warps active, issue active) + its parity test
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/time_cfg.py 3 5 > gpurun_out/c3_time.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/c3_launches.csv python scripts/time_cfg.py 3 1 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c3" > gpurun_out/c3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c3_pytest.log
