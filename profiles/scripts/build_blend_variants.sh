# blend.cu register-cap variants -> profiles/variants/libtgs_<name>.so (A/B with profiles/ab_variants.sh)
set -e
cd "$(dirname "$0")/../../paper_2501_14534_b200/csrc"
make -s
mkdir -p ../../profiles/variants
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
build() {  # name, defines...
  name=$1; shift
  nvcc $F "$@" -c blend.cu -o /tmp/blend_$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64 \
       -o ../../profiles/variants/libtgs_$name.so $(ls build/*.o | grep -v build/blend.o) /tmp/blend_$name.o
}
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  build $name $(for d in ${defs//,/ }; do echo -D$d; done)
done
