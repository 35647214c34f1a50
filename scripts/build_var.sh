# usage: bash scripts/build_var.sh <name> "<extra nvcc flags>" [quant source]  -> build/<name>/libdctf_var.so
# (measurement variants of csrc/quant.cu linked with the product objects; load with DCTF_LIB_PATH)
set -e
cd "$(dirname "$0")/.."
NAME=$1; FLAGS=$2; SRC=${3:-paper_1710_07193_b200/csrc/quant.cu}
mkdir -p build/$NAME
make -s build/capi.o build/coef.o build/fused.o build/tc.o build/ozaki.o build/spatial.o build/host.o build/plan.o
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3 \
  --expt-relaxed-constexpr -I paper_1710_07193_b200/csrc $FLAGS -c -o build/$NAME/quant.o $SRC
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/$NAME/libdctf_var.so \
  build/capi.o build/coef.o build/fused.o build/tc.o build/ozaki.o build/spatial.o build/$NAME/quant.o build/host.o build/plan.o -ldl
