# scratch iteration: full GPU parity + per-config timing
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
for c in 1 2 3 4 5; do timeout 200 python scripts/time_cfg.py $c 5; done > gpurun_out/it_time.log 2>&1
