# A/B of kernel-variant builds (profiles/variants/*.so, built with -D overrides of the
# launch bounds) on the c3 bench: step/s, render FPS and the per-launch stage times.
# Usage (repo root): bash profiles/ab_variants.sh profiles/variants/a.so profiles/variants/b.so ...  (default build first and last)
# Building a variant (here: loss.cu with -DNAME=VALUE; the kernel reads the macro):
#   cd paper_2501_14534_b200/csrc && make
#   F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
#      -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"   # + -fmad=false for preprocess.cu
#   nvcc $F -DNAME=VALUE -c loss.cu -o /tmp/loss_v.o
#   nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared \
#        -Xlinker -rpath,/usr/local/cuda/lib64 -o ../../profiles/variants/libtgs_v.so \
#        $(ls build/*.o | grep -v build/loss.o) /tmp/loss_v.o
for v in "" "$@" ""; do
  TGS_LIB=$(test -n "$v" && realpath $v) python bench.py > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);s=d['stages'];print('${v:-default}', d['value'], d['render_fps'], *(k+'='+str(s[k]['ms_per_launch']) for k in ('preprocess_fwd','blend_fwd','loss','blend_bwd','preprocess_bwd')))"
done
