"""Does tcgen05.mma kind::tf32 truncate or round its fp32 inputs?  One pass (hi*hi) on raw fp32
operands (debug flag: no split) vs float64 sums of truncated / round-to-nearest-away inputs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_06528_b200 import push

def tf32(x, mode):
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    if mode == "rna":
        u = u + 0x1000
    return (u & 0xFFFFE000).astype(np.uint32).view(np.float32).astype(np.float64)

rng = np.random.default_rng(0)
M, N, K = 128, 128, 256
A = rng.standard_normal((1, M, K)).astype(np.float32)
B = rng.standard_normal((1, N, K)).astype(np.float32)
C = push.gemm3xtf32(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), False, False, M, N, K,
                    passes=1 | (1 << 8), b_split=True).double().cpu().numpy()
for mode in ("trunc", "rna"):
    ref = tf32(A[0], mode) @ tf32(B[0], mode).T
    print(mode, "max abs diff", np.abs(C[0] - ref).max())
