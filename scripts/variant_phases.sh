#!/bin/bash
# bench.py per-class phases of build variants in .variants/ (experiments only; restores the product library):
#   bash scripts/variant_phases.sh <tag> "<configs>" <variant> ...
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
LIB=paper_2306_06528_b200/libpush_b200.so
cp $LIB /tmp/lib_product.so
for V in product "$@"; do
  if [ "$V" != product ]; then cp .variants/lib_$V.so $LIB; else cp /tmp/lib_product.so $LIB; fi
  for C in $CFGS; do
    timeout 300 python bench.py --config $C --no-cpu-baseline --steps 20 --warmup 5 > $OUT/bench_${C}_$V.json 2>&1
    python - "$OUT/bench_${C}_$V.json" "$V" <<'PY'
import json, sys
try:
    j = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ph = {k: round(v["ms_per_step"], 4) for k, v in j["phases"].items()}
    print(sys.argv[2], j["config"]["workload"][:3], round(j["value"], 1), round(j["ms_per_step"], 4), ph)
except Exception as e:
    print(sys.argv[1], "no line", e)
PY
  done
done
cp /tmp/lib_product.so $LIB
