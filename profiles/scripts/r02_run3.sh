TGS_LIB=$PWD/profiles/variants/libtgs_count.so timeout 600 python profiles/exact_pairs.py > gpurun_out/exact_pairs_v1.json 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v3.json 2>gpurun_out/bench_v3.err
TGS_EXACT=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v3_noexact.json 2>gpurun_out/bench_v3n.err
