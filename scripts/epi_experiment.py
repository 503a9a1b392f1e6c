"""C2 forward shape, store vs fused forward epilogue, 1-CTA vs pair kernel (run under ncu for times)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_06528_b200 import push
M, N, K, batch = 8192, 256, 256, 16
A = (0.5 * torch.randn(batch, M, K, device="cuda")).tanh()
B = torch.rand(batch, N, K, device="cuda") / 8 - 1 / 16
for flags in (0, 32, 96):
    for _ in range(4):
        push.gemm3xtf32(A, B, False, False, M, N, K, passes=3 | (flags << 8), b_split=True)
    torch.cuda.synchronize()
