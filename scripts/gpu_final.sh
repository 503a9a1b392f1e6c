#!/bin/bash
# Round-end evidence in one gpurun call: GPU tests, smoke, default bench (S1, with CPU baseline), every
# config's bench line, reference arm, ncu launch list + full capture of the S1 step, and the per-class
# DRAM traffic probe of every config (profiles/traffic_<cfg>.json is summarised on the dev host).
#   gpurun --timeout 3000 -- 'bash scripts/gpu_final.sh r01g'
TAG=${1:-final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt 2>&1
python -c "from paper_2306_06528_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2>> $OUT/bench.err
for C in C1 C2 C3 C4 C5 C5b; do
  timeout 600 python bench.py --config $C --no-cpu-baseline > $OUT/bench_$C.json 2>> $OUT/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'gemm3xtf32|svgd_update|dist_|gram_|output_stream|finalize' \
  -s 40 -c 8 -o $OUT/prof python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > $OUT/ncu_full.log 2>&1
for C in C2 C3 C4 C5 S1; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none \
    --csv --log-file gpurun_out/traffic_$C.csv python scripts/traffic_probe.py --config $C > $OUT/traffic_$C.log 2>&1
done
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; head -c 400 $OUT/bench.json; echo; head -c 300 $OUT/bench_reference.json
