cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 240 -k "c2 or top_stream or fused or c1" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 2 2 2; do timeout 120 python scripts/time_cfg.py $c 10 >> gpurun_out/time_cfg.log 2>&1; done
