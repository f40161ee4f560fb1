# lazy long levels: parity on the long-path tests, timings lazy vs two-pass
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "
import paper_1602_02740_b200 as tg, json
for n in (1<<20, 1<<24):
    d = tg.plan_describe(n, 1, B=4 if n == 1<<20 else 16, long_count=0)
    print(json.dumps([(l['B'], l['count'], l['n'], l['long'], l['res'], l['lazy']) for l in d['levels']]), d['workspace_bytes'])
" > gpurun_out/q_plan.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checks.py -m gpu -q -x --timeout 600 -rf -k "long or c4 or c5 or stage or t16 or b32 or squaring or ntt or wrapper or signed or sharded or unbalanced or workspace" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
for c in 4 5; do timeout 300 python scripts/time_cfg.py $c 5 >> gpurun_out/q_time.log 2>&1; TOOM_LAZY=0 timeout 300 python scripts/time_cfg.py $c 3 >> gpurun_out/q_time.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launches_c4.csv python scripts/time_cfg.py 4 1 > gpurun_out/q_ncu_c4.log 2>&1
