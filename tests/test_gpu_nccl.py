"""The NCCL exchange path on one GPU: PUSH_FORCE_NCCL=1 gives every context a single-rank NCCL
communicator, so the comm-stream Theta all-gather, the G all-gather, the loss gather and the CUDA-graph
capture of NCCL calls all run for real; the results must be bit-identical to the NCCL-free path.
(The multi-rank NCCL data path needs several GPUs; host-side multi-process logic is covered by
tests/test_dist_gloo.py.)"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from inputs import WORKLOADS, synth
from paper_2306_06528_b200 import push
w = WORKLOADS["C1"]
out = {{}}
for mode in ("eager", "graph"):
    ctx = push.Context(push.make_config(w.n_particles, list(w.dims), max_batch=w.batch, seed=3, step_size=1e-2))
    loss = torch.empty(w.n_particles, device="cuda")
    for t in range(4):
        x, y = synth.workload_batch(w, t)
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        if mode == "eager":
            ctx.particle_grads(xd, yd, loss)
            ctx.svgd_step()
        else:
            ctx.step_graph(xd, yd, loss)
    out[mode] = (ctx.gather("theta"), ctx.gather("grad"), ctx.gather("loss"), ctx.gather("dist"))
np.savez({path!r}, **{{f"{{m}}_{{i}}": a for m, v in out.items() for i, a in enumerate(v)}})
"""


def _run(tmp_path, force):
    path = str(tmp_path / f"nccl{force}.npz")
    env = dict(os.environ, PUSH_FORCE_NCCL=str(force))
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, path=path)], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(path)


def test_single_rank_nccl_path_bit_identical(tmp_path):
    a = _run(tmp_path, 0)
    b = _run(tmp_path, 1)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
