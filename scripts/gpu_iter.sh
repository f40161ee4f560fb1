cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
for r in 1 2; do
for v in base nopeel; do
  if [ $v = base ]; then L=; else L=variants/libtoomgpu_$v.so; fi
  for c in 1 2 3; do echo -n "$v " >> gpurun_out/it_time.log; TOOM_LIB=$L timeout 300 python scripts/time_cfg.py $c 20 >> gpurun_out/it_time.log 2>&1; done
done; done
