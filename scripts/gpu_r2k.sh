cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/k_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k_pytest_gpu.log
for c in 4 5; do timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/k_time.log 2>&1; done
for c in 4 5; do TOOM_MULTI_CH4_NS=99 timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/k_time_ch16.log 2>&1; done
timeout 300 python scripts/time_cfg.py 5 1 > gpurun_out/k_plain5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k_launches_c5.csv python scripts/time_cfg.py 5 1 > gpurun_out/k_ncu_c5.log 2>&1
