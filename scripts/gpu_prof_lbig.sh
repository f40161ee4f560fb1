# ncu full set of k_lbig2 (C5's matrix-form Toom-16 interpolation), one launch
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_lbig2" -c 2 -o gpurun_out/prof_lbig python scripts/time_cfg.py 5 1 > gpurun_out/prof_lbig.log 2>&1
