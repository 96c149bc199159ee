set -x
export TGS_PARITY_REPORT=gpurun_out/parity_r02_v2.json
timeout 1800 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -40 > gpurun_out/pytest_gpu_v2.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v2.json 2>gpurun_out/bench_v2.err
