cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf -x -k "long or c4 or c5 or stage or signed or sharded or check or verify" > gpurun_out/e_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/e_pytest_gpu.log
for c in 4 5; do timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/e_time.log 2>&1; done
timeout 300 python scripts/time_cfg.py 4 1 > gpurun_out/e_plain4.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e_launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/e_ncu_c4.log 2>&1
