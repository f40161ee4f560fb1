# scratch iteration: long/lazy parity + C4/C5 timing
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checks.py -m gpu -q -x -k "lazy or c4 or c5 or long or t16 or squaring or b32 or wrapper or stage or signed or verify" > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
for c in 4 5; do timeout 200 python scripts/time_cfg.py $c 5; done > gpurun_out/it_time.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it_launches.csv python scripts/time_cfg.py 4 1 > /dev/null 2>&1
