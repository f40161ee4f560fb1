cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "" variants/libtoomgpu_ch8.so variants/libtoomgpu_ch32.so; do echo "lib $v"; TOOM_LIB=$v timeout 200 python scripts/time_cfg.py 4 5; TOOM_LIB=$v timeout 200 python scripts/time_cfg.py 5 2; done > gpurun_out/v.log 2>&1
