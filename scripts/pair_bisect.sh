#!/bin/bash
# run the CTA-pair GEMM under debug flag combinations, one process each (a fault kills the context)
for F in 0 2 4 6 16 20 22; do
  timeout 60 python - <<PY 2>&1 | tail -1
import torch, sys
sys.path.insert(0, ".")
from paper_2306_06528_b200 import push
M, N, K = 300, 256, 128
A = torch.randn(1, M, K, device="cuda"); B = torch.randn(1, N, K, device="cuda")
try:
    C = push.gemm3xtf32(A, B, False, False, M, N, K, passes=3 | ($F << 8), b_split=False)
    torch.cuda.synchronize()
    ref = (A.double() @ B.double().transpose(1, 2))
    print("flags=$F ok maxerr", float((C.double() - ref).abs().max()))
except Exception as e:
    print("flags=$F FAIL", str(e)[:120])
PY
done
