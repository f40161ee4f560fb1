# round 2, second GPU pass: parity + checks after the check fixes, bench, probe + T16 long-op profiles
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/b_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/b_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/b_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/b_bench.log
timeout 300 python scripts/probe_run.py > gpurun_out/b_probe.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_probe -c 2 -o gpurun_out/b_prof_probe python scripts/probe_run.py > gpurun_out/b_ncu_probe.log 2>&1
timeout 300 python scripts/time_cfg.py 5 1 > gpurun_out/b_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_long_op -s 520 -c 3 -o gpurun_out/b_prof_t16op python scripts/time_cfg.py 5 1 > gpurun_out/b_ncu_t16.log 2>&1
