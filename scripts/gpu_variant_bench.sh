#!/bin/bash
# NEXT-2 measurement: bench lines with --variant paper next to the canonical ones
TAG=${1:-varb}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "from paper_2306_06528_b200 import build; build.build()" > $OUT/build.log 2>&1
for c in ${CFGS:-C2 C3 C4 C5}; do
  for v in canonical paper; do
    timeout 300 python bench.py --config $c --variant $v --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_${c}_$v.json 2> $OUT/bench_${c}_$v.err
  done
done
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob(os.environ.get("OUT", "gpurun_out/x") + "/*.json")):
    pass
PY
for f in $OUT/bench_*.json; do python -c "
import json,sys
l=json.loads(open('$f').read().strip().splitlines()[-1])
ph=l['phases']
print('$f', round(l['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in ph.items() if k in ('distances','bandwidth_k','svgd_update')})
" 2>&1 | tail -1; done
