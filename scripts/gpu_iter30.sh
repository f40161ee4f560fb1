cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 240 -k "long or c4 or c5 or stage or sharded" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for tp in 64 1000000; do echo "twopass=$tp" >> gpurun_out/time_cfg.log; for c in 4 5; do TOOM_TWO_PASS_TILES=$tp timeout 200 python scripts/time_cfg.py $c 3 >> gpurun_out/time_cfg.log 2>&1; done; done
