cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do
for v in base h5 h11 h13; do
  if [ $v = base ]; then L=; else L=variants/libtoomgpu_$v.so; fi
  echo -n "$v " >> gpurun_out/it_time.log
  TOOM_LIB=$L timeout 300 python scripts/time_cfg.py 2 20 >> gpurun_out/it_time.log 2>&1
done; done
