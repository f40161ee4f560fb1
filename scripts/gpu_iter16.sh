cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in default r64 r72; do
  echo "variant=$v" >> gpurun_out/time_cfg.log
  if [ $v = default ]; then L=""; else L="$GRAFT_REPO_ROOT/build_variants/libtoomgpu_$v.so"; fi
  for c in 2 4; do TOOM_LIB=$L timeout 120 python scripts/time_cfg.py $c 10 >> gpurun_out/time_cfg.log 2>&1; done
done
