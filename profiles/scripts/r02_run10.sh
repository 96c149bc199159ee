export TGS_PARITY_REPORT=gpurun_out/parity_r02_v12.json
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/pytest_gpu_v12.log
timeout 600 python bench.py > gpurun_out/bench_v12.json 2>gpurun_out/bench_v12.err
mkdir -p /tmp/ncu
python profiles/profile_step.py > gpurun_out/ps.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -f -o /tmp/ncu/view_r02 python profiles/profile_step.py > gpurun_out/ncu_view.log 2>&1
python profiles/profile_train.py > gpurun_out/pt.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_preprocess_bwd|k_adam|k_exact" -f -o /tmp/ncu/step_r02 python profiles/profile_train.py > gpurun_out/ncu_step.log 2>&1
python profiles/ncu_summary.py --prefix r02 /tmp/ncu/view_r02.ncu-rep /tmp/ncu/step_r02.ncu-rep > gpurun_out/ncu_summary.log 2>&1
cp profiles/r02_ncu_summary.txt profiles/r02_ncu_traffic.json gpurun_out/ 2>/dev/null
ncu -i /tmp/ncu/view_r02.ncu-rep --page source --csv -k regex:k_blend_bwd16w > gpurun_out/r02_blend_bwd_source.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
du -sh gpurun_out; ls -la gpurun_out | head -40
