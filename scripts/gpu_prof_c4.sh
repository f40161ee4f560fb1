# ncu full set of every launch of ONE C4 product (the 21 launches after the warm-up product), long-vector kernels included
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 200 python scripts/time_cfg.py 4 1 > gpurun_out/prof_c4.pre.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --launch-skip 21 -c 21 -o gpurun_out/prof_c4 python scripts/time_cfg.py 4 1 > gpurun_out/prof_c4.log 2>&1
