cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/h_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/h_pytest_gpu.log
for c in 4 5; do timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/h_time.log 2>&1; done
timeout 900 python bench.py > gpurun_out/h_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/h_bench.log
