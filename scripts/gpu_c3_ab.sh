# C3 A/B: split-multiplier row kernel vs the generic one; parity on the C3 tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checks.py -q -x -k "c3 or p8 or check or fault" > gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
for v in 1 0 1; do echo "split=$v" >> gpurun_out/ab_time.log; TOOM_P8_ROWS_SPLIT=$v timeout 300 python scripts/time_cfg.py 3 5 >> gpurun_out/ab_time.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/ab_c3_launches.csv python scripts/time_cfg.py 3 1 > /dev/null 2>&1
