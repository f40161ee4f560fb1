cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in default e96 e80; do
  echo "variant=$v" >> gpurun_out/time_cfg.log
  if [ $v = default ]; then L=""; else L="$GRAFT_REPO_ROOT/build_variants/libtoomgpu_$v.so"; fi
  for c in 3 4; do TOOM_LIB=$L timeout 120 python scripts/time_cfg.py $c 5 >> gpurun_out/time_cfg.log 2>&1; done
done
for m in 7 3 1 0; do echo "mask=$m" >> gpurun_out/time_cfg.log; TOOM_DBG_FUSED_MASK=$m timeout 120 python scripts/time_cfg.py 2 10 >> gpurun_out/time_cfg.log 2>&1; done
