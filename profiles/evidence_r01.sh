set -x
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_v2.log
python bench.py > gpurun_out/v15a.json 2>gpurun_out/v15a.err
python bench.py > gpurun_out/v15b.json 2>gpurun_out/v15b.err
python bench.py --config c4 > gpurun_out/c4_v10.json 2>gpurun_out/c4_v10.err
python bench.py --config c5 > gpurun_out/c5_v5.json 2>gpurun_out/c5_v5.err
python profile_step.py > gpurun_out/ps.log 2>&1 && ncu --set full --clock-control none --import-source on --profile-from-start off -f -o gpurun_out/view_v2 python profile_step.py > gpurun_out/ncu_view.log 2>&1
python profile_train.py > gpurun_out/pt.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_preprocess_bwd|k_adam" -f -o gpurun_out/step_v2 python profile_train.py > gpurun_out/ncu_step.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bl.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_v2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
