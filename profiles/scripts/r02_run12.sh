mkdir -p /tmp/ncu
for v in default p1; do
  if [ $v = default ]; then L=""; else L=$PWD/profiles/variants/libtgs_$v.so; fi
  TGS_LIB=$L timeout 900 ncu --set full --clock-control none -k regex:k_blend_bwd16 --profile-from-start off -f -o /tmp/ncu/bwd_$v python profiles/profile_step.py > gpurun_out/ncu_bwd_$v.log 2>&1
  ncu -i /tmp/ncu/bwd_$v.ncu-rep --page raw --csv > gpurun_out/ncu_bwd_$v.csv 2>/dev/null
  ncu -i /tmp/ncu/bwd_$v.ncu-rep --page details > gpurun_out/ncu_bwd_$v.txt 2>/dev/null
done
