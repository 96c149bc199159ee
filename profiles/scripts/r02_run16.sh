timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_gpu_v19.log
bash profiles/scripts/ab.sh v19 profiles/variants/libtgs_b5.so profiles/variants/libtgs_b3.so env:TGS_EXACT=0 > gpurun_out/ab_v19.txt 2>&1
