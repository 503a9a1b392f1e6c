"""Does the tcgen05 fp32 accumulator round to nearest or truncate?  Positive-only products over a
long K, accumulated entirely in TMEM (debug flag 8, one pass, raw tf32-exact inputs): a truncating
accumulator shows a negative bias ~ -K/2 ulp; round-to-nearest shows ~sqrt(K) ulp noise."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_06528_b200 import push

rng = np.random.default_rng(1)
for K in (256, 1024, 8192):
    M, N = 128, 128
    # tf32-exact positive inputs so products are exact in fp32; only the accumulation rounds
    A = (rng.integers(1, 1024, (1, M, K)) / 1024.0).astype(np.float32)
    B = (rng.integers(1, 1024, (1, N, K)) / 1024.0).astype(np.float32)
    ref = A[0].astype(np.float64) @ B[0].astype(np.float64).T
    for flags, name in ((8, "whole-K in TMEM"), (0, "promoted every 128")):
        C = push.gemm3xtf32(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), False, False, M, N, K,
                            passes=1 | (flags << 8), b_split=True).double().cpu().numpy()[0]
        rel = (C - ref) / ref
        print(f"K={K:5d} {name:20s} mean rel err {rel.mean():+.3e}  max |rel| {np.abs(rel).max():.3e}")
