# ncu full set of every launch of ONE C4 product (the 21 launches after the warm-up product), long-vector kernels included;
# summaries are written on the box (the reports are too large to bring back)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 200 python scripts/time_cfg.py 4 1 > gpurun_out/prof_c4.pre.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --launch-skip 21 -c 21 -o /tmp/prof_c4 -f python scripts/time_cfg.py 4 1 > gpurun_out/prof_c4.log 2>&1
python scripts/ncu_raw_summary.py /tmp/prof_c4.ncu-rep > gpurun_out/prof_c4_raw_summary.csv
ncu -i /tmp/prof_c4.ncu-rep --page details --csv > gpurun_out/prof_c4_details.csv 2>/dev/null
for k in k_lz_eval_last k_lz_interp k_lz_eval k_lz_fin; do python scripts/sass_hot.py /tmp/prof_c4.ncu-rep $k > gpurun_out/prof_c4_sass_hot_$k.txt 2>&1; done
