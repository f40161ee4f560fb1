cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TOOM_SLOW=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 1400 -k "c5_full_oracle or c5_full or c4_single" -rA > gpurun_out/c5_oracle.log 2>&1; echo "rc=$?" >> gpurun_out/c5_oracle.log
