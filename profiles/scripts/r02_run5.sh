export TGS_PARITY_REPORT=gpurun_out/parity_r02_v5.json
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -30 > gpurun_out/pytest_gpu_v5.log
bash profiles/scripts/ab.sh v5 profiles/variants/libtgs_s0c68.so profiles/variants/libtgs_s0c78.so profiles/variants/libtgs_s1.so profiles/variants/libtgs_s1c68.so env:TGS_EXACT=0 > gpurun_out/ab_v5.txt 2>&1
TGS_LIB=$PWD/profiles/variants/libtgs_count.so timeout 600 python profiles/exact_pairs.py > gpurun_out/exact_pairs_v2.json 2>&1
