#!/bin/bash
# bench every workload once (no CPU baseline) — sanity + numbers for DESIGN/BASELINE tables
TAG=${1:-cfg}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "from paper_2306_06528_b200 import build; build.build()" > $OUT/build.log 2>&1
for C in ${CONFIGS:-C1 C2 C3 C4 C5 S1}; do
  timeout 600 python bench.py --config $C --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > $OUT/bench_$C.json 2> $OUT/bench_$C.err
  echo "$C exit $?"; tail -2 $OUT/bench_$C.err
done
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob(os.environ.get("OUT", "gpurun_out/cfg") + "/bench_*.json")):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no json", e); continue
    r = j["roofline"]
    print(f"{j['config']['workload'][:3]} {j['value']:10.1f} ps/s  {j['ms_per_step']:8.3f} ms/step  {r['kernel']:28s} {r['frac']:.3f} {r.get('all_gemm_tflops', 0):6.1f}TF  upd {r.get('svgd_update_hbm_frac', 0):.2f}")
    print("     ", {k: round(v['ms_per_step'], 3) for k, v in j['phases'].items()})
PY
