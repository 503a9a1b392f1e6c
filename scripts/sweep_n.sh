#!/bin/bash
# time per step vs particle count at fixed networks ("quadratic scaling" claim, on B200)
OUT=gpurun_out/${1:-sweep}
mkdir -p $OUT
python -c "from paper_2306_06528_b200 import build; build.build()" > $OUT/build.log 2>&1
for C in C4 C2; do
  for N in 8 16 32 64 128 256 512; do
    if [ $C = C2 ] && [ $N -gt 128 ]; then continue; fi
    timeout 300 python bench.py --config $C --n-particles $N --steps 10 --warmup 3 --no-cpu-baseline > $OUT/${C}_$N.json 2>/dev/null
  done
done
python - <<'PY'
import json, glob, os
out = os.environ.get("OUT", "gpurun_out/sweep")
for f in sorted(glob.glob(out + "/*.json")):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    ph = {k: round(v["ms_per_step"], 4) for k, v in j["phases"].items() if k in ("distances", "bandwidth_k", "svgd_update")}
    print(os.path.basename(f), j["config"]["n_particles"], round(j["ms_per_step"], 4), ph)
PY
