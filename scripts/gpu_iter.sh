# scratch iteration: C2 parity (all modes) + checks, per-mode C2 timing, launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checks.py -m gpu -q -x -k "c2 or fault or check or c1" > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
for m in "" "TOOM_DEFERRED_BOTTOM=0" "TOOM_C2_CLS=0"; do echo "env $m"; env $m timeout 120 python scripts/time_cfg.py 2 10; done > gpurun_out/it_time.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it_launches.csv python scripts/time_cfg.py 2 1 > /dev/null 2>&1
