cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in 7 3 1 0; do echo "mask=$m" >> gpurun_out/time_cfg.log; TOOM_DBG_FUSED_MASK=$m timeout 120 python scripts/time_cfg.py 2 10 >> gpurun_out/time_cfg.log 2>&1; done
timeout 300 ncu --set full --clock-control none --import-source on -k "regex:k_interp_top_smem|k_fused_bottom" -c 2 -o gpurun_out/prof_c2_r3 python scripts/prof_c2.py 1 > gpurun_out/ncu_full.log 2>&1
