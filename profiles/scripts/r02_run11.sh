timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "golden or c1_gradients or deterministic or multiview" 2>&1 | tail -3 > gpurun_out/pytest_q_v13.log
bash profiles/scripts/ab.sh v13 profiles/variants/libtgs_p1.so profiles/variants/libtgs_m4.so profiles/variants/libtgs_m3.so profiles/variants/libtgs_m6.so > gpurun_out/ab_v13.txt 2>&1
