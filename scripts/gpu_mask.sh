# fused-bottom phase shares on C2 (TOOM_DBG_FUSED_MASK: bit0 products, bit1 rows, bit2 recomposition)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for m in 0 1 3 7; do echo "mask $m"; TOOM_DBG_FUSED_MASK=$m timeout 120 python scripts/time_cfg.py 2 10; done > gpurun_out/mask.log 2>&1
