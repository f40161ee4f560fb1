# two-pass long-op executor: parity + timings vs the look-back executor
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf -x > gpurun_out/c_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c_pytest_gpu.log
for c in 4 5; do timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/c_time.log 2>&1; done
for c in 4 5; do TOOM_LONG_LOOKBACK=1 timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/c_time_lookback.log 2>&1; done
timeout 300 python scripts/time_cfg.py 4 1 > gpurun_out/c_plain4.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/c_ncu_c4.log 2>&1
