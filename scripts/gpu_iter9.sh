cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 2 4 5; do timeout 120 python scripts/time_cfg.py $c 3 >> gpurun_out/time_cfg.log 2>&1; done
for m in 512 1024; do TOOM_LONG_MIN_N=$m timeout 120 python scripts/time_cfg.py 4 3 >> gpurun_out/time_cfg_minn.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/ncu_c4.log 2>&1
