cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python scripts/c5_sharded.py --n 65536 --steps 2 --warmup 1 > gpurun_out/c5_sharded.log 2>&1; echo "c5s rc=$?" >> gpurun_out/c5_sharded.log
