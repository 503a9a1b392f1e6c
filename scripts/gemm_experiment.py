"""Time the product GEMM kernel on the C2 forward / weight-gradient shapes under debug variants
(bit 0: skip the in-smem hi/lo split, bit 1: skip the epilogue math/stores, bit 2: skip the MMAs)
to locate the bottleneck.  GPU only; run under `ncu --metrics gpu__time_duration.sum` for clean
kernel times (the printed CUDA-event times include the debug entry's host-side scratch handling)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_06528_b200 import push

shapes = {"fwd_bsplit": (8192, 256, 256, 0, 0, 1, 16), "fwd_bpair": (8192, 256, 256, 0, 0, 0, 16),
          "bwd_bsplit": (8192, 256, 256, 0, 1, 1, 16), "bwd_bpair": (8192, 256, 256, 0, 1, 0, 16),
          "wgrad_ks1024": (256, 256, 1024, 1, 1, 1, 128)}
variants = [(3, 0), (3, 2), (3, 4), (3, 6), (1, 0)]
for name, (M, N, K, amn, bmn, bsplit, batch) in shapes.items():
    A = torch.randn(batch, *((K, M) if amn else (M, K)), device="cuda")
    B = torch.randn(batch, *((K, N) if bmn else (N, K)), device="cuda")
    for passes, flags in variants:
        for _ in range(4):
            push.gemm3xtf32(A, B, amn, bmn, M, N, K, passes=passes | (flags << 8), b_split=bool(bsplit))
        torch.cuda.synchronize()
        print(name, passes, flags, flush=True)
