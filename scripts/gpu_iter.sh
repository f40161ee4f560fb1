cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
for c in 3 4; do for s in 1 0; do echo -n "st=$s " >> gpurun_out/it_time.log; TOOM_ITS_STATIC=$s timeout 300 python scripts/time_cfg.py $c 10 >> gpurun_out/it_time.log 2>&1; done; done
