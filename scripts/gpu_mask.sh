# scratch: C5 with the multi-output ops at 4 limbs per thread from NS sources up (TOOM_MULTI_CH4_NS)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/ch4_*.log
for ns in 1048576 16 8 4; do echo "ns $ns" >> gpurun_out/ch4_time.log; TOOM_MULTI_CH4_NS=$ns timeout 300 python scripts/time_cfg.py 5 3 >> gpurun_out/ch4_time.log 2>&1; done
TOOM_MULTI_CH4_NS=16 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ch4_c5_launches.csv python scripts/time_cfg.py 5 1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/ch4_c5_launches.csv 40 > gpurun_out/ch4_c5_summary.log 2>&1
