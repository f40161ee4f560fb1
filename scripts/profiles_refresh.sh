# copy the evidence of scripts/gpu_evidence.sh (gpurun_out/ev_*) into profiles/ (round tag $1, default r01)
cd "$(dirname "$0")/.."
T=${1:-r01}
python scripts/traffic_json.py gpurun_out/ev_prof_c2.ncu-rep > profiles/traffic.json
grep '^{' gpurun_out/ev_bench.log > profiles/${T}_bench.jsonl
grep '^{' gpurun_out/ev_ref.log > profiles/${T}_reference.jsonl
cp gpurun_out/ev_launches.csv profiles/${T}_c2_bench_launches.csv
python scripts/launch_summary.py gpurun_out/ev_launches.csv 10 > profiles/${T}_c2_bench_launches_summary.txt
cp gpurun_out/ev_launches_c4.csv profiles/${T}_c4_launches.csv
python scripts/launch_summary.py gpurun_out/ev_launches_c4.csv 40 > profiles/${T}_c4_launches_summary.txt
grep '^{' gpurun_out/ev_time_cfg.log > profiles/${T}_time_cfg.jsonl
ncu -i gpurun_out/ev_prof_c2.ncu-rep --page details --csv > profiles/${T}_c2_ncu_full_details.csv 2>/dev/null
ncu -i gpurun_out/ev_prof_c2.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keys=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum']
idx=[h.index(k) for k in keys if k in h]
print(','.join(h[i] for i in idx)); print(','.join(r[1][i] for i in idx))
for x in r[2:]: print(','.join('\"'+x[i]+'\"' if ',' in x[i] else x[i] for i in idx))
" > profiles/${T}_c2_ncu_raw_summary.csv
for k in k_fused_dc k_interp_top_cls k_eval_top_v4; do python scripts/sass_hot.py gpurun_out/ev_prof_c2.ncu-rep $k > profiles/${T}_sass_hot_$k.txt 2>&1; done
cp gpurun_out/ev_pytest_gpu.log profiles/${T}_pytest_gpu.log
cp gpurun_out/ev_launches_c5.csv profiles/${T}_c5_launches.csv 2>/dev/null && python scripts/launch_summary.py gpurun_out/ev_launches_c5.csv 40 > profiles/${T}_c5_launches_summary.txt
