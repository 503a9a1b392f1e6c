"""S1/C3 forward shapes through the pair kernel: plain store vs fused forward epilogue (tanh / identity)
vs no epilogue (debug flag), CUDA-event timed (median of 10).  Isolates the epilogue's share."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_06528_b200 import push
for (M, N, K, batch) in ((8192, 512, 512, 64), (8192, 1024, 1024, 16), (8192, 256, 256, 16)):
    A = (0.5 * torch.randn(batch, M, K, device="cuda")).tanh()
    B = torch.rand(batch, N, K, device="cuda") / 8 - 1 / 16
    fl = 2.0 * M * N * K * batch
    for name, flags in (("store", 0), ("fwd-tanh", 32), ("fwd-id", 96), ("no-epi", 2), ("no-mma", 4), ("no-mma-no-epi", 6)):
        ts = []
        for _ in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            push.gemm3xtf32(A, B, False, False, M, N, K, passes=3 | (flags << 8), b_split=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts[2:])[len(ts[2:]) // 2]
        print(f"M{M} N{N} K{K} b{batch} {name:14s} {t*1e3:8.1f} us  {fl/t/1e9:7.1f} TF/s useful")
