mkdir -p /tmp/ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_blend_(bwd16p|fwd16w)" --profile-from-start off -f -o /tmp/ncu/blend python profiles/profile_step.py > gpurun_out/ncu_blend.log 2>&1
ncu -i /tmp/ncu/blend.ncu-rep --page source --csv --print-source sass -k regex:k_blend_bwd16p > gpurun_out/bwd16p_sass.csv 2>gpurun_out/src.err
ncu -i /tmp/ncu/blend.ncu-rep --page source --csv --print-source sass -k regex:k_blend_fwd16w > gpurun_out/fwd16w_sass.csv 2>>gpurun_out/src.err
ls -la gpurun_out/*sass.csv
