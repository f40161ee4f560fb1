# ncu full set of C5's top-level kernels (Toom-16 evaluation k_lmulti2<1,16>, matrix-form interpolation k_lbig2 / k_lmulti2<0,16>), first product
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:k_lbig2|k_lmulti2" -c 22 -o /tmp/prof_c5top -f python scripts/time_cfg.py 5 1 > gpurun_out/prof_c5top.log 2>&1
python scripts/ncu_raw_summary.py /tmp/prof_c5top.ncu-rep > gpurun_out/prof_c5top_raw_summary.csv
ncu -i /tmp/prof_c5top.ncu-rep --page details --csv > gpurun_out/prof_c5top_details.csv 2>/dev/null
for i in 0 1; do python scripts/sass_hot.py /tmp/prof_c5top.ncu-rep k_lbig2 $i > gpurun_out/prof_c5top_sass_hot_k_lbig2_$i.txt 2>&1; python scripts/sass_hot.py /tmp/prof_c5top.ncu-rep k_lmulti2 $i > gpurun_out/prof_c5top_sass_hot_k_lmulti2_$i.txt 2>&1; done
ncu -i /tmp/prof_c5top.ncu-rep -k regex:k_lbig2 --page source --csv --print-source sass > gpurun_out/prof_c5top_lbig2_source.csv 2>/dev/null; gzip -f gpurun_out/prof_c5top_lbig2_source.csv
ncu -i /tmp/prof_c5top.ncu-rep -k regex:k_lbig2 --page source --csv --print-source cuda > gpurun_out/prof_c5top_lbig2_cuda.csv 2>/dev/null; gzip -f gpurun_out/prof_c5top_lbig2_cuda.csv
