#!/bin/bash
# quick check + ncu: launch list of a 2-step bench and a full capture of the GEMMs and output kernel
#   gpurun --timeout 1800 -- 'bash scripts/gpu_prof.sh tag [config]'
TAG=${1:-prof}
CFG=${2:-C2}
OUT=gpurun_out/$TAG
bash scripts/gpu_quick.sh $TAG
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gemm3xtf32|output_fused|finalize' \
  -s 14 -c 16 -o $OUT/prof python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_full.log 2>&1
tail -3 $OUT/ncu_full.log
