cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 240 -k "long or c4 or c5 or stage" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in default lo1 lo3; do
  echo "variant=$v" >> gpurun_out/time_cfg.log
  if [ $v = default ]; then L=""; else L="$GRAFT_REPO_ROOT/build_variants/libtoomgpu_$v.so"; fi
  for c in 4 5; do TOOM_LIB=$L timeout 200 python scripts/time_cfg.py $c 3 >> gpurun_out/time_cfg.log 2>&1; done
done
