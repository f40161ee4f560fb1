# scratch iteration: C3 parity + timing
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checks.py -m gpu -q -x -k "c3 or p8 or ragged or 8-" > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
for m in 1 0; do TOOM_EVAL_P8=$m timeout 200 python scripts/time_cfg.py 3 5; done > gpurun_out/it_time.log 2>&1
