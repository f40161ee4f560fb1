cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/time_cfg.py 5 1 > gpurun_out/plain_c5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_long_op" --launch-skip 30 -c 2 -o gpurun_out/prof_t16op python scripts/time_cfg.py 5 1 > gpurun_out/ncu_t16.log 2>&1
