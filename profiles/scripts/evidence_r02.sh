# The round-2 evidence set (files copied into profiles/ as r02_*): run from the repo root
# under gpurun.  Each ncu capture runs only after the same command exited 0 without ncu.
# The .ncu-rep captures are summarised on the box and deleted (gpurun copies back <= 64 MiB).
set -x
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_final.log
python bench.py > gpurun_out/bench_final.json 2>gpurun_out/bench_final.err
python bench.py --impl reference > gpurun_out/bench_ref_final.json 2>gpurun_out/bench_ref_final.err
python bench.py --config c4 > gpurun_out/c4_final.json 2>gpurun_out/c4_final.err
python bench.py --config c5 > gpurun_out/c5_final.json 2>gpurun_out/c5_final.err
for n in 2 4 8; do for dp in gaussians zero; do python bench.py --rank-share $n --dp $dp > gpurun_out/rank_share_${dp}_$n.json 2>gpurun_out/rank_share_${dp}_$n.err; done; done
python profiles/rank_share_trace.py 8 gaussians > gpurun_out/r02_rank_share_trace_gaussians_8.txt 2>&1
python profiles/rank_share_trace.py 8 zero > gpurun_out/r02_rank_share_trace_zero_8.txt 2>&1
python profiles/step_host_latency.py gaussians > gpurun_out/r02_step_host_latency_gaussians.txt 2>&1
python profiles/profile_step.py > gpurun_out/ps.log 2>&1 && ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"^(k_|tgs)" -f -o gpurun_out/view_final python profiles/profile_step.py > gpurun_out/ncu_view.log 2>&1
python profiles/profile_train.py > gpurun_out/pt.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_preprocess_bwd|k_adam|k_exact|k_preprocess_fwd" -f -o gpurun_out/step_final python profiles/profile_train.py > gpurun_out/ncu_step.log 2>&1
python profiles/ncu_summary.py --prefix r02 gpurun_out/view_final.ncu-rep gpurun_out/step_final.ncu-rep > gpurun_out/ncu_summary.log 2>&1
cp profiles/r02_ncu_summary.txt profiles/r02_ncu_traffic.json gpurun_out/
for k in bwd16p fwd16w; do
  ncu -i gpurun_out/view_final.ncu-rep --page source --csv --kernel-name regex:$k --print-source sass > gpurun_out/src_$k.csv 2>/dev/null
  (echo "ncu -i <c3 view capture, profiles/scripts/evidence_r02.sh> --page source --csv --kernel-name regex:$k --print-source sass | python profiles/sass_classes.py"; python profiles/sass_classes.py gpurun_out/src_$k.csv) > gpurun_out/r02_blend_${k}_sass_classes.txt
  rm -f gpurun_out/src_$k.csv
done
rm -f gpurun_out/*.ncu-rep
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bl.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
