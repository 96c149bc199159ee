timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_gpu_v20.log
bash profiles/scripts/ab.sh v20 env:TGS_BWD_CHUNKS=1 env:TGS_BWD_CHUNKS=2 env:TGS_BWD_CHUNKS=8 > gpurun_out/ab_v20.txt 2>&1
