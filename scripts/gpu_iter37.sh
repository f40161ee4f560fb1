cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for ss in 2 1 3; do echo "split=$ss" >> gpurun_out/time_cfg.log; TOOM_SPLIT_STREAMS=$ss timeout 200 python scripts/time_cfg.py 2 10 >> gpurun_out/time_cfg.log 2>&1; TOOM_SPLIT_STREAMS=$ss timeout 200 python scripts/time_cfg.py 3 5 >> gpurun_out/time_cfg.log 2>&1; done
