# scratch iteration: C4 / lazy / C5 parity and timings, C4 launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/it_*.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "c4 or lazy or long or c5 or t16" > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
for c in 4 4 5; do timeout 300 python scripts/time_cfg.py $c 5 >> gpurun_out/it_time.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it_c4_launches.csv python scripts/time_cfg.py 4 1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/it_c4_launches.csv 40 > gpurun_out/it_c4_summary.log 2>&1
