#!/bin/bash
# quick GPU check: gemm unit tests, parity tests, smoke, short bench (each under its own timeout)
#   gpurun --timeout 1500 -- 'bash scripts/gpu_quick.sh tag'
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > $OUT/gpu.txt
python -c "from paper_2306_06528_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 200 python -m pytest tests/test_gpu_gemm.py -x -q > $OUT/gemm.log 2>&1; echo "exit $?" >> $OUT/gemm.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q > $OUT/parity.log 2>&1; echo "exit $?" >> $OUT/parity.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "exit $?" >> $OUT/smoke.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
PUSH_GEMM_PAIR=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "grads or c2" > $OUT/parity_pair.log 2>&1; tail -1 $OUT/parity_pair.log
grep -E "^FAILED|passed|failed" $OUT/gemm.log | head -20; grep -E "^FAILED|passed|failed|^E " $OUT/parity.log | head -30; tail -2 $OUT/smoke.log; cat $OUT/bench.json | head -c 3000; tail -5 $OUT/bench.err
