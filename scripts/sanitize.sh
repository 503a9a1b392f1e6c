#!/bin/bash
# compute-sanitizer memcheck / racecheck over small GPU cases (TMA/tcgen05 kernels included)
OUT=gpurun_out/${1:-sanitize}
mkdir -p $OUT
python -c "from paper_2306_06528_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "grads_match_oracle or step_from_set_grads or sharding or step_graph" > $OUT/memcheck.log 2>&1; echo "memcheck exit $?" >> $OUT/memcheck.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_gemm.py -q -x \
  -k "512 or 300" > $OUT/memcheck_gemm.log 2>&1; echo "memcheck_gemm exit $?" >> $OUT/memcheck_gemm.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "grads_match_oracle and dims0" > $OUT/racecheck.log 2>&1; echo "racecheck exit $?" >> $OUT/racecheck.log
for f in memcheck memcheck_gemm racecheck; do tail -n 4 $OUT/$f.log; done
