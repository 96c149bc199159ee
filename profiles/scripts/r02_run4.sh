export TGS_PARITY_REPORT=gpurun_out/parity_r02_v4.json
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -30 > gpurun_out/pytest_gpu_v4.log
bash profiles/scripts/ab.sh v4 profiles/variants/libtgs_b6.so profiles/variants/libtgs_b7.so profiles/variants/libtgs_b6f8.so profiles/variants/libtgs_b7f8.so env:TGS_EXACT=0 > gpurun_out/ab_v4.txt 2>&1
