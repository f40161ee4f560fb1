# profile the two-pass long kernels on C4's level-4 interpolation rows
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/time_cfg.py 4 1 > gpurun_out/d_plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lmulti2 -s 50 -c 2 -o gpurun_out/d_prof_lmulti2 python scripts/time_cfg.py 4 1 > gpurun_out/d_ncu.log 2>&1
