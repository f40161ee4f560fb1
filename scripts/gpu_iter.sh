# scratch iteration: C4/C5 parity and per-config timings
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/it_*.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c4 or lazy or long_path or c5_shape" > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
for c in 4 5; do timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/it_time.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it_c4_launches.csv python scripts/time_cfg.py 4 1 > /dev/null 2>&1
