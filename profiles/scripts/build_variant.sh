# one translation unit rebuilt with -D defines -> profiles/variants/libtgs_<name>.so (A/B via TGS_LIB)
# usage: bash profiles/scripts/build_variant.sh <name> <file.cu> [DEFINE[=V] ...]
set -e
name=$1; src=$2; shift 2
cd "$(dirname "$0")/../../paper_2501_14534_b200/csrc"
make -s
mkdir -p ../../profiles/variants
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
obj=build/${src%.cu}.o
nvcc $F $(for d in "$@"; do echo -D$d; done) -c $src -o /tmp/var_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64 \
     -o ../../profiles/variants/libtgs_$name.so $(ls build/*.o | grep -v "^$obj$") /tmp/var_$name.o
