cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/time_cfg.py 4 1 > gpurun_out/s_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k "regex:k_lz_interp|k_lz_eval_last" -c 3 -o gpurun_out/s_prof_c4 python scripts/time_cfg.py 4 1 > gpurun_out/s_ncu_c4.log 2>&1
ls -la gpurun_out >> gpurun_out/s_ncu_c4.log
