# Build an experimental variant of libtoomgpu.so with extra nvcc flags:
#   bash scripts/build_variant.sh NAME -DFLAG ...   -> variants/libtoomgpu_NAME.so
# (select it at run time with TOOM_LIB=variants/libtoomgpu_NAME.so)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
python -c "from paper_1602_02740_b200.build import generate; generate()"
mkdir -p variants
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared \
  -I include "$@" -o variants/libtoomgpu_$name.so paper_1602_02740_b200/csrc/*.cu
