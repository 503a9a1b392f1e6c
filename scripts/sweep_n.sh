#!/bin/bash
# step time vs particle count at fixed d (PAPER.md:355's "quadratic in the number of particles"):
#   gpurun -- 'bash scripts/sweep_n.sh <tag>'   ->  gpurun_out/<tag>/sweep.txt
OUT=gpurun_out/${1:-sweep}
mkdir -p $OUT
python -c "from paper_2306_06528_b200 import build; build.build()" > $OUT/build.log 2>&1
for spec in "C2 8 16 32 64 128" "C4 8 16 32 64 128 256 512"; do
  set -- $spec; C=$1; shift
  for n in "$@"; do
    timeout 300 python bench.py --config $C --n-particles $n --no-cpu-baseline --steps 10 --warmup 3 > $OUT/${C}_$n.json 2>> $OUT/err.log
    python - "$OUT/${C}_$n.json" $C $n >> $OUT/sweep.txt <<'PY'
import json, sys
j = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph = j["phases"]
kp = sum(ph[k]["ms_per_step"] for k in ("distances", "bandwidth_k", "svgd_update") if k in ph)
print(f"| {sys.argv[2]} | {sys.argv[3]} | {j['ms_per_step']:.4f} | {j['value']:,.0f} | {kp:.4f} |")
PY
  done
done
cat $OUT/sweep.txt
