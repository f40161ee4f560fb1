# lazy levels: debug products, full GPU suite, timings, C4/C5 launch lists
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/lazy_debug.py > gpurun_out/r_dbg.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/r_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r_pytest.log
for c in 4 5; do timeout 300 python scripts/time_cfg.py $c 5 >> gpurun_out/r_time.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r_launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/r_ncu_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r_launches_c5.csv python scripts/time_cfg.py 5 1 > gpurun_out/r_ncu_c5.log 2>&1
