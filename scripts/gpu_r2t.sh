# f2: tensor-core base case parity + timing (bounded: a descriptor bug could spin the mbarrier wait)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_core" > gpurun_out/t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_pytest.log
timeout 180 python scripts/time_tc_base.py 5 > gpurun_out/t_time.log 2>&1; echo "rc=$?" >> gpurun_out/t_time.log
