for v in "" profiles/variants/libtgs_noinl.so profiles/variants/libtgs_minb5.so; do
  TGS_LIB=$v python profiles/exc_ab.py > gpurun_out/exc_ab_$(basename ${v:-default}).json 2>&1
done
