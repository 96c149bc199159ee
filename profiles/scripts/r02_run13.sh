export TGS_PARITY_REPORT=gpurun_out/parity_r02_v14.json
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -25 > gpurun_out/pytest_gpu_v14.log
bash profiles/scripts/ab.sh v14 env:TGS_TRAIN_NATIVE=0 > gpurun_out/ab_v14.txt 2>&1
timeout 900 python bench.py --config c5 > gpurun_out/c5_v14.json 2>gpurun_out/c5_v14.err
TGS_TRAIN_NATIVE=0 timeout 900 python bench.py --config c5 > gpurun_out/c5_v14py.json 2>gpurun_out/c5_v14py.err
