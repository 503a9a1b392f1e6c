"""g error vs the oracle (inf-rel per particle, max) for C2-, S1- and C3-shaped networks at the current
PUSH_GEMM_CHUNK / PUSH_GEMM_CHUNK_FB (promotion chunk of all / of the forward-backward GEMMs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from inputs import synth
from oracle import mlp as omlp
from paper_2306_06528_b200 import push
tag = "chunk_fb=%s" % os.environ.get("PUSH_GEMM_CHUNK_FB", "-")
for dims, B in (([2, 256, 256, 256, 256, 1], 2048), ([3, 512, 512, 512, 512, 512, 1], 2048),
                ([3, 1024, 1024, 1024, 1024, 1], 1024), ([2, 2048, 2048, 2048, 1], 512)):
    x, y = synth.batch("advection" if dims[0] == 2 else "burgers", B, dims[0], dims[-1], step=3)
    ctx = push.Context(push.make_config(2, dims, max_batch=B, seed=2))
    th = ctx.gather("theta")
    ctx.particle_grads(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    g = ctx.gather("grad").astype(np.float64)
    G, _ = omlp.grads_all(th, dims, x, y)
    err = max(np.abs(g[i] - G[i]).max() / np.abs(G[i]).max() for i in range(2))
    print(tag, dims[1], len(dims) - 2, "B", B, "inf-rel g err %.3e" % err, flush=True)
