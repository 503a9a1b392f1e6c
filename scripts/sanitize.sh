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
# the shared-memory kernels added in session 3: streaming output layer (slab ring), staged update,
# n <= 8 distances, column-group finalize / distance reduction
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "(grads_match_oracle and (dims7 or dims12 or dims14 or dims15)) or (step_from_set_grads and (33-777 or 64-2048 or 5-4099 or 100-96))" \
  > $OUT/racecheck2.log 2>&1; echo "racecheck2 exit $?" >> $OUT/racecheck2.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "(grads_match_oracle and (dims12 or dims13 or dims14 or dims15 or dims16)) or (step_from_set_grads and (4-3333 or 6-20000 or 300-64 or 130-999 or 160-3000 or 96-1537 or 64-2048))" \
  > $OUT/memcheck2.log 2>&1; echo "memcheck2 exit $?" >> $OUT/memcheck2.log
# Gram distances + tensor-core update across a loopback group (n = 128, P = 1/2/4)
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "sharding and 128" > $OUT/memcheck3.log 2>&1; echo "memcheck3 exit $?" >> $OUT/memcheck3.log
for f in memcheck memcheck_gemm racecheck racecheck2 memcheck2 memcheck3; do tail -n 4 $OUT/$f.log; done
# round 2: the Gram-form distances (gram.cu, n = 33..256), the streaming update (upd.cu, n = 33..64),
# both through the d-sharded panels too
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "(step_from_set_grads and (33-777 or 64-2048 or 100-96 or 160-3000)) or (clustered and (64-0.1 or 256))" \
  > $OUT/memcheck_r02.log 2>&1; echo "memcheck_r02 exit $?" >> $OUT/memcheck_r02.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "step_from_set_grads and (33-777 or 64-2048 or 160-3000)" > $OUT/racecheck_r02.log 2>&1; echo "racecheck_r02 exit $?" >> $OUT/racecheck_r02.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_dshard.py -q -x \
  -k "dims5" > $OUT/memcheck_r02_dshard.log 2>&1; echo "memcheck_r02_dshard exit $?" >> $OUT/memcheck_r02_dshard.log
for f in memcheck_r02 racecheck_r02 memcheck_r02_dshard; do tail -n 3 $OUT/$f.log; done
