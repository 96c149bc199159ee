timeout 900 python bench.py --config c5 > gpurun_out/c5_v15.json 2>gpurun_out/c5_v15.err
timeout 900 python bench.py --config c4 > gpurun_out/c4_v15.json 2>gpurun_out/c4_v15.err
timeout 900 python bench.py --rank-share 8 --steps 5 > gpurun_out/rs8_v15.json 2>gpurun_out/rs8_v15.err
timeout 900 python bench.py --rank-share 2 --steps 5 > gpurun_out/rs2_v15.json 2>gpurun_out/rs2_v15.err
timeout 900 python bench.py --rank-share 4 --steps 5 > gpurun_out/rs4_v15.json 2>gpurun_out/rs4_v15.err
