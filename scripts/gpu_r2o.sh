cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -rf -k "ntt or wrapper" > gpurun_out/o_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/o_pytest_gpu.log
for a in "4 0" "4 4" "4 16" "5 16" "5 4" "5 0"; do timeout 300 python scripts/time_ntt.py $a 3 >> gpurun_out/o_time.log 2>&1; done
