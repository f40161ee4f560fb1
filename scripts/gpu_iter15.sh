cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for m in 7 3; do echo "mask=$m" >> gpurun_out/time_cfg.log; TOOM_DBG_FUSED_MASK=$m timeout 120 python scripts/time_cfg.py 2 10 >> gpurun_out/time_cfg.log 2>&1; done
for c in 4; do timeout 120 python scripts/time_cfg.py $c 5 >> gpurun_out/time_cfg.log 2>&1; done
python -c "
import sys; sys.path.insert(0,'.')
import paper_1602_02740_b200 as tg, torch
torch.cuda.init()
print('wide', tg.probe_limb_products()); print('chain', tg.probe_carry_chain())" >> gpurun_out/time_cfg.log 2>&1
