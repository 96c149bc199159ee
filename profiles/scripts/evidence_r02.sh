# The round-2 evidence set (files copied into profiles/ as r02_*): run from the repo root
# under gpurun.  Each ncu capture runs only after the same command exited 0 without ncu.
set -x
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_final.log
python bench.py > gpurun_out/bench_final.json 2>gpurun_out/bench_final.err
python bench.py --impl reference > gpurun_out/bench_ref_final.json 2>gpurun_out/bench_ref_final.err
python bench.py --config c4 > gpurun_out/c4_final.json 2>gpurun_out/c4_final.err
for n in 2 4 8; do python bench.py --rank-share $n > gpurun_out/rank_share_$n.json 2>gpurun_out/rank_share_$n.err; done
python profiles/profile_step.py > gpurun_out/ps.log 2>&1 && ncu --set full --clock-control none --import-source on --profile-from-start off -f -o gpurun_out/view_final python profiles/profile_step.py > gpurun_out/ncu_view.log 2>&1
python profiles/profile_train.py > gpurun_out/pt.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_preprocess_bwd|k_adam|k_exact|k_preprocess_fwd" -f -o gpurun_out/step_final python profiles/profile_train.py > gpurun_out/ncu_step.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bl.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
