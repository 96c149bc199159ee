# blend backward variants on one c3 view set (profiles/exc_ab.py): TGS_LIB per variant
for v in "" "$@"; do
  TGS_LIB=$v python profiles/exc_ab.py > gpurun_out/exc_ab_$(basename ${v:-default}).json 2>&1
done
