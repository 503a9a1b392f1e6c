#!/bin/bash
# NEXT-2 check: variant parity tests + the canonical parity suite + a short bench (regression)
#   gpurun --timeout 1200 -- 'bash scripts/gpu_variant.sh tag'
TAG=${1:-var}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "from paper_2306_06528_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 400 python -m pytest tests/test_gpu_variant.py tests/test_gpu_dshard.py -q > $OUT/variant.log 2>&1; echo "exit $?" >> $OUT/variant.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nccl.py -q > $OUT/parity.log 2>&1; echo "exit $?" >> $OUT/parity.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
grep -E "^FAILED|passed|failed|^E " $OUT/variant.log | head -40; grep -E "^FAILED|passed|failed|^E " $OUT/parity.log | head -20; head -c 400 $OUT/bench.json; tail -3 $OUT/bench.err
