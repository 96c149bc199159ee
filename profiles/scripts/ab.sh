# quick A/B of library variants on the c3 bench (no CPU baseline): prints step/s and stage times
# usage: bash profiles/scripts/ab.sh <tag> [lib.so | env:VAR=VAL] ...
tag=$1; shift
for v in "" "$@"; do
  if [[ "$v" == env:* ]]; then e=${v#env:}; lib=""; else e=""; lib=$(test -n "$v" && realpath $v); fi
  env $e TGS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err
  python -c "import json;d=json.loads(open('gpurun_out/ab_$tag.json').read().strip().splitlines()[-1]);s=d['stages'];print('${v:-default}', d['value'], d['e2e']['value'], d['render_fps'], *(k+'='+str(s[k]['ms_per_launch']) for k in ('preprocess_fwd','blend_fwd','loss','blend_bwd','preprocess_bwd')))" || tail -5 gpurun_out/ab_$tag.err
done
