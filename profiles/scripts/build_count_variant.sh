# libtgs with the float64 decision counter (-DTGS_COUNT_EXACT) -> profiles/variants/libtgs_count.so
set -e
cd "$(dirname "$0")/../../paper_2501_14534_b200/csrc"
make -s
mkdir -p ../../profiles/variants
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
nvcc $F -DTGS_COUNT_EXACT -c blend.cu -o /tmp/blend_count.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64 \
     -o ../../profiles/variants/libtgs_count.so $(ls build/*.o | grep -v build/blend.o) /tmp/blend_count.o
