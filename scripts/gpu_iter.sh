# scratch iteration: stage exports / sharded path
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi.py -q -x -k "stage or sharded or signed or abi" > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
