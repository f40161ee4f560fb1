cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 240 -k "long or c4 or c5 or stage" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for mc in 1073741824 50000 8000; do echo "maxcount=$mc" >> gpurun_out/time_cfg.log; for c in 4 5; do TOOM_LONG_MAX_COUNT=$mc timeout 200 python scripts/time_cfg.py $c 3 >> gpurun_out/time_cfg.log 2>&1; done; done
