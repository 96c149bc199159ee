# A/B of kernel-variant builds (profiles/variants/*.so, built with -D overrides of the
# launch bounds) on the c3 bench: step/s, render FPS and the per-launch stage times.
# Usage: bash profiles/ab_variants.sh variants/a.so variants/b.so ...  (default build first and last)
for v in "" "$@" ""; do
  TGS_LIB=$(test -n "$v" && realpath $v) python bench.py > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);s=d['stages'];print('${v:-default}', d['value'], d['render_fps'], *(k+'='+str(s[k]['ms_per_launch']) for k in ('preprocess_fwd','blend_fwd','loss','blend_bwd','preprocess_bwd')))"
done
