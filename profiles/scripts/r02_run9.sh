export TGS_PARITY_REPORT=gpurun_out/parity_r02_v9.json
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -40 > gpurun_out/pytest_gpu_v9.log
timeout 600 python bench.py > gpurun_out/bench_v9.json 2>gpurun_out/bench_v9.err
