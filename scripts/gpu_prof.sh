# ncu full set of the C2 kernels (current build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_fused_dc|k_interp_top|k_eval_top_v4" -c 3 -o gpurun_out/prof_it python scripts/prof_c2.py 1 > gpurun_out/prof_it.log 2>&1
