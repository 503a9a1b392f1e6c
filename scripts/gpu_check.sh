#!/bin/bash
# Iteration check on one GPU: selected GPU tests and short bench lines of the given configs.
#   gpurun --timeout 1500 -- 'bash scripts/gpu_check.sh <tag> "<pytest -k expr or empty>" "C2 S1"'
TAG=${1:-check}
KEXPR=${2:-}
CFGS=${3:-"C2 S1"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "from paper_2306_06528_b200 import build; build.build()" > $OUT/build.log 2>&1
if [ -n "$KEXPR" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -k "$KEXPR" > $OUT/pytest.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest.log 2>&1
fi
echo "pytest exit $?" >> $OUT/pytest.log
for C in $CFGS; do
  timeout 600 python bench.py --config $C --no-cpu-baseline --steps 10 --warmup 3 > $OUT/bench_$C.json 2> $OUT/bench_$C.err
done
tail -5 $OUT/pytest.log
for C in $CFGS; do python - "$OUT/bench_$C.json" <<'PY'
import json, sys
try:
    j = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ph = {k: round(v["ms_per_step"], 4) for k, v in j["phases"].items()}
    print(j["config"]["workload"][:3], round(j["value"], 1), "ms/step", round(j["ms_per_step"], 4), ph)
except Exception as e:
    print(sys.argv[1], "no line", e)
PY
done
