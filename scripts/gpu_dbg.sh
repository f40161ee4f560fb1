cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out variants
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -I oldsrc/include -o variants/libtoomgpu_head.so oldsrc/paper_1602_02740_b200/csrc/*.cu > gpurun_out/dbg_build.log 2>&1
echo "== head" > gpurun_out/dbg3.log; TOOM_LIB=variants/libtoomgpu_head.so python scripts/lazy_debug.py >> gpurun_out/dbg3.log 2>&1
