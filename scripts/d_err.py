"""Max relative error of the GPU distances against the float64 oracle (Gram form accuracy probe).
    python scripts/d_err.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from inputs import synth
from oracle import svgd as osvgd
from paper_2306_06528_b200 import push

for n, spread in [(64, 1e-1), (64, 1e-2), (128, 1e-2), (256, 1e-3), (64, None), (128, None)]:
    d = 20000
    Th = synth.clustered_theta(n, d, seed=n, spread=spread) if spread else synth.random_theta(n, d, seed=n, scale=0.2)
    G = synth.random_grads(n, d, seed=5)
    ctx = push.Context(push.make_config(n, [d - 1, 1], max_batch=1, step_size=0.05), theta0=Th)
    ctx.set_grads(torch.from_numpy(G).cuda())
    ctx.svgd_step()
    _, info = osvgd.svgd_step(Th, G, 0.05)
    D = ctx.gather("dist")
    off = ~np.eye(n, dtype=bool)
    print(n, spread, "max rel D err %.3e" % np.max(np.abs(D[off] - info["D"][off]) / info["D"][off]))
