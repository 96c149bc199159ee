# c5 survival vs the held-out subset's opacity boost (bench.py schedule_c5, TGS_C5_BOOST)
for b in 0 1 2 4; do
  TGS_C5_BOOST=$b timeout 600 python bench.py --config c5 > gpurun_out/c5_boost_$b.json 2> gpurun_out/c5_boost_$b.err
done
