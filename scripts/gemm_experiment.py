"""Time the product GEMM kernel on the C2 forward / backward / weight-gradient shapes under
debug variants (passes, skip-transform) to locate the bottleneck.  GPU only."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_06528_b200 import push

def t(fn, it=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it

res = {}
for name, (M, N, K, amn, bmn, bsplit) in {"fwd": (8192, 256, 256, 0, 0, 0), "bwd": (8192, 256, 256, 0, 1, 0),
                                          "wgrad_ks1024": (256, 256, 1024, 1, 1, 1)}.items():
    batch = 16 if name != "wgrad_ks1024" else 128
    A = torch.randn(batch, *((K, M) if amn else (M, K)), device="cuda")
    B = torch.randn(batch, *((K, N) if bmn else (N, K)), device="cuda")
    for passes in (3, 1):
        for skip in (0, 1):
            ms = t(lambda: push.gemm3xtf32(A, B, amn, bmn, M, N, K, passes=passes | (skip << 8), b_split=bool(bsplit)))
            fl = 2.0 * M * N * K * batch
            res[f"{name} passes={passes} skip_split={skip}"] = {"us": ms * 1e3, "useful_TF": fl / ms / 1e9}
for k, v in res.items():
    print(f"{k:40s} {v['us']:8.1f} us  {v['useful_TF']:6.1f} TF")
