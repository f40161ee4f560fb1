# re-entry check: full GPU suite, bench line, per-config timings, C4/C5 launch lists
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/p_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/p_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/p_bench.log
for c in 1 2 3 4 5; do timeout 300 python scripts/time_cfg.py $c 5 >> gpurun_out/p_time.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/p_ncu_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches_c5.csv python scripts/time_cfg.py 5 1 > gpurun_out/p_ncu_c5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches_c3.csv python scripts/time_cfg.py 3 1 > gpurun_out/p_ncu_c3.log 2>&1
