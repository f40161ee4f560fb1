# scratch iteration: C2 + C3 parity and per-config timings
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/it_*.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checks.py -q -x -k "c2 or c3 or p8 or check or fault" > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
for c in 2 3; do timeout 300 python scripts/time_cfg.py $c 5 >> gpurun_out/it_time.log 2>&1; done
