set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export TGS_PARITY_REPORT=gpurun_out/parity_r02_v1.json
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -60 > gpurun_out/pytest_gpu_v1.log
timeout 600 python bench.py > gpurun_out/bench_v1.json 2>gpurun_out/bench_v1.err
timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/bench_v1_s20.json 2>gpurun_out/bench_v1_s20.err
ls -la gpurun_out
