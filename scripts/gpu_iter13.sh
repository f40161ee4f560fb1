cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in 7 3 1 0; do echo "mask=$m" >> gpurun_out/time_cfg.log; TOOM_DBG_FUSED_MASK=$m timeout 120 python scripts/time_cfg.py 2 10 >> gpurun_out/time_cfg.log 2>&1; done
