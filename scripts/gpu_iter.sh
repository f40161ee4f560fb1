# scratch GPU iteration: parity tests + C2 step timing (edit freely)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
for r in 1 2 3; do timeout 300 python scripts/time_cfg.py 2 20 >> gpurun_out/it_time.log 2>&1; done
