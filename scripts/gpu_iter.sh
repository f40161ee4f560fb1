# scratch iteration: C2 + C4 parity + timing
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checks.py -m gpu -q -x -k "c2 or fault or check or lazy or c4 or c5_shape" > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
for c in 2 2 4; do timeout 200 python scripts/time_cfg.py $c 20; done > gpurun_out/it_time.log 2>&1
