cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 1 2 3 4; do timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/time_cfg.log 2>&1; done
timeout 300 python scripts/prof_c2.py 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_interp_top_rows|k_fused_bottom|k_eval_top_rows" -c 3 -o gpurun_out/prof_c2_full python scripts/prof_c2.py 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
