cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
for m in 0 24000 200000 0 24000 200000; do echo -n "m=$m " >> gpurun_out/it_time.log; TOOM_EVAL_PTS_MAX_COUNT=$m timeout 300 python scripts/time_cfg.py 4 5 >> gpurun_out/it_time.log 2>&1; done
for m in 0 24000 200000; do echo -n "m=$m " >> gpurun_out/it_time.log; TOOM_EVAL_PTS_MAX_COUNT=$m timeout 300 python scripts/time_cfg.py 3 10 >> gpurun_out/it_time.log 2>&1; done
for m in 0 24000; do echo -n "m=$m " >> gpurun_out/it_time.log; TOOM_EVAL_PTS_MAX_COUNT=$m timeout 300 python scripts/time_cfg.py 5 2 >> gpurun_out/it_time.log 2>&1; done
