for v in "" profiles/variants/libtgs_bwd16minb7.so profiles/variants/libtgs_bwd16minb8.so profiles/variants/libtgs_fwd16minb10.so profiles/variants/libtgs_adj4.so ""; do
  TGS_LIB=$(test -n "$v" && realpath $v) python bench.py > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);s=d['stages'];print('${v:-default}', d['value'], d['render_fps'], s['blend_fwd']['ms_per_launch'], s['blend_bwd']['ms_per_launch'], s['loss']['ms_per_launch'])"
done
