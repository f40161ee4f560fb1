cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf -x -k "long or c4 or c5 or stage or signed or sharded or check or verify or rows" > gpurun_out/g_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g_pytest_gpu.log
for c in 4 5; do timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/g_time.log 2>&1; done
for c in 4 5; do TOOM_RES=0 timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/g_time_nores.log 2>&1; done
for c in 4 5; do TOOM_RES_MIN_N=1000 timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/g_time_res1000.log 2>&1; done
