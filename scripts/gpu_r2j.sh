cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/time_cfg.py 5 1 > gpurun_out/j_plain5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_launches_c5.csv python scripts/time_cfg.py 5 1 > gpurun_out/j_ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lbig2 -s 8 -c 2 -o gpurun_out/j_prof_lbig2 python scripts/time_cfg.py 5 1 > gpurun_out/j_ncu_lbig.log 2>&1
