# scratch iteration: C3 / ragged / rows parity and timings, C3 launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/it_*.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "c3 or ragged or rows or p8 or top_stream or long_vs_short or squaring or c1 or c2_slice" > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
for c in 3 3 4; do timeout 300 python scripts/time_cfg.py $c 10 >> gpurun_out/it_time.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it_c3_launches.csv python scripts/time_cfg.py 3 1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/it_c3_launches.csv 40 > gpurun_out/it_c3_summary.log 2>&1
