#!/bin/bash
# One build -> measure iteration: GPU tests, benches of CONFIGS, and an ncu full capture of the kernels
# matching KREGEX on config PCFG (skip with KREGEX="").
#   gpurun --timeout 1800 -- 'CONFIGS="C2 C5" PCFG=C5 KREGEX="dist_small|svgd_update" bash scripts/gpu_iter.sh tag'
TAG=${1:-iter}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > $OUT/gpu.txt
python -c "from paper_2306_06528_b200 import build; build.build()" > $OUT/build.log 2>&1
if [ -z "${NOTEST:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $OUT/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $OUT/pytest_gpu.log
fi
for C in ${CONFIGS:-C2}; do
  timeout 600 python bench.py --config $C --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} \
    > $OUT/bench_$C.json 2> $OUT/bench_$C.err
done
if [ -n "${KREGEX:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${NCU_SKIP:-0} -c ${NCU_COUNT:-8} \
    -o $OUT/prof python bench.py --config ${PCFG:-C2} --steps 1 --warmup 1 --no-cpu-baseline --no-graph > $OUT/ncu_full.log 2>&1
  tail -3 $OUT/ncu_full.log
fi
tail -3 $OUT/pytest_gpu.log 2>/dev/null
python - "$OUT" <<'PY'
import json, glob, sys
for f in sorted(glob.glob(sys.argv[1] + "/bench_*.json")):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no json", e); continue
    r = j["roofline"]
    print(f"{j['config']['workload'][:3]} {j['value']:10.1f} ps/s  {j['ms_per_step']:8.3f} ms/step  {r['kernel']:28s} {r['frac']:.3f} {r.get('all_gemm_tflops', 0):6.1f}TF  upd {r.get('svgd_update_hbm_frac', 0):.2f} clk {j['clocks']['sm_mhz']}")
    print("     ", {k: round(v['ms_per_step'], 3) for k, v in j['phases'].items()})
PY
