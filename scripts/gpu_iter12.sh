cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for kb in 113 75 56 38; do echo "kb=$kb" >> gpurun_out/time_cfg.log; TOOM_ITS_SMEM_KB=$kb timeout 120 python scripts/time_cfg.py 2 10 >> gpurun_out/time_cfg.log 2>&1; done
