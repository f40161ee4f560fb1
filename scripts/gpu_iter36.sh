cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/sanitize_small.py > gpurun_out/sanitize_small.log 2>&1
for mn in 2048 4098 16386; do echo "minn=$mn" >> gpurun_out/time_cfg.log; for c in 4 5; do TOOM_LONG_MIN_N=$mn timeout 200 python scripts/time_cfg.py $c 3 >> gpurun_out/time_cfg.log 2>&1; done; done
