# round 2, first GPU pass: parity + checks, bench line, probe + C4 long-kernel profiles
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi > gpurun_out/a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/a_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/a_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/a_bench.log
timeout 300 python scripts/probe_run.py > gpurun_out/a_probe.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_probe -c 2 -o gpurun_out/a_prof_probe python scripts/probe_run.py > gpurun_out/a_ncu_probe.log 2>&1
timeout 300 python scripts/time_cfg.py 4 3 > gpurun_out/a_c4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_long_multi -s 20 -c 4 -o gpurun_out/a_prof_c4multi python scripts/time_cfg.py 4 1 > gpurun_out/a_ncu_c4.log 2>&1
