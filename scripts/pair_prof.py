import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_06528_b200 import push
M, N, K, batch = 8192, 256, 256, 16
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
A = torch.randn(batch, M, K, device="cuda"); B = torch.randn(batch, N, K, device="cuda")
for _ in range(3):
    push.gemm3xtf32(A, B, False, False, M, N, K, passes=3 | (flags << 8), b_split=True)
torch.cuda.synchronize()
