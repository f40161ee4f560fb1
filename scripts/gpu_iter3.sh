cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "long or c4 or c5 or stage or top_stream" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 2 4 5; do timeout 300 python scripts/time_cfg.py $c 5 >> gpurun_out/time_cfg.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_interp_top_smem" -c 1 -o gpurun_out/prof_interp_smem python scripts/prof_c2.py 1 > gpurun_out/ncu_full.log 2>&1
