# round evidence: parity tests, bench line, reference arm, launch list, full ncu of the C2 kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/ev_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/ev_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/ev_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/ev_ref.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c4 --no-c5 > gpurun_out/ev_bench_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c4 --no-c5 > gpurun_out/ev_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_eval_top_v4|k_fused_bottom|k_fused_dc|k_interp_top" -c 3 -o gpurun_out/ev_prof_c2 python scripts/prof_c2.py 1 > gpurun_out/ev_ncu_full.log 2>&1
for c in 1 2 3 4 5; do timeout 300 python scripts/time_cfg.py $c 5 >> gpurun_out/ev_time_cfg.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/ev_ncu_c4.log 2>&1
nvidia-smi > gpurun_out/ev_smi.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c5.csv python scripts/time_cfg.py 5 1 > gpurun_out/ev_ncu_c5.log 2>&1
