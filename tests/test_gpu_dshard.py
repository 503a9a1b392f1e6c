"""NEXT-4 on one GPU: the d-sharded kernel phase (push_config.exchange = DSHARD, include/push.h).

Rank q owns whole distance splits = a column range of every particle; the kernel phase runs on
column panels after an all-to-all transpose and the updated columns go back to the row owners.
Every element sees the splits, sums and update arithmetic of the all-gather path, so Theta, D, h and
the losses must be BIT-identical to it for P = 1, 2, 4, 8 (loopback transport of
push_init_local_group) and through the NCCL send/recv path (PUSH_FORCE_NCCL=1 single-rank
communicator).  The all-gather path itself is pinned to the oracle by tests/test_gpu_parity.py; one
oracle step is re-checked here too."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import synth  # noqa: E402
from oracle import mlp as omlp  # noqa: E402
from oracle import svgd as osvgd  # noqa: E402
from paper_2306_06528_b200 import push  # noqa: E402

from .gpu_util import rel_err  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _run(dims, n, B, P, exchange, steps=3, seed=9):
    x, y = synth.batch("gauss", B, dims[0], dims[-1], 1)
    xd, yd = _dev(x), _dev(y)
    cfg = push.make_config(n, dims, max_batch=B, step_size=1e-2, seed=seed, exchange=exchange)
    ctxs = push.local_group(cfg, P) if P > 1 else [push.Context(cfg)]
    for t in range(steps):
        for c in ctxs:
            c.particle_grads(xd, yd)
        for c in ctxs:
            c.svgd_step()
    return (ctxs[0].gather("theta"), ctxs[-1].gather("loss"), ctxs[0].gather("dist"), ctxs[-1].gather("h"),
            ctxs[-1].gather("kernel"))


@pytest.mark.parametrize("dims,n,B", [
    ([2, 64, 64, 1], 8, 256),
    ([1, 32, 32, 1], 4, 256),
    ([2, 256, 256, 1], 16, 512),      # many splits, ragged split counts per rank
    ([1, 8, 1], 8, 64),               # d = 25: one split, ranks 1.. own no columns
    ([3, 40, 24, 2], 24, 100),        # thin layers, ld padding inside the last rank's panel
    ([1, 32, 32, 1], 64, 128),        # n = 64: the Gram-form partials (NP = 64) on column panels
])
def test_dshard_bit_identical_to_allgather(dims, n, B):
    base = _run(dims, n, B, 1, "allgather")
    for P in (1, 2, 4, 8):
        if n % P:
            continue
        r = _run(dims, n, B, P, "dshard")
        for k, (a, b) in enumerate(zip(r[:4], base[:4])):
            assert np.array_equal(a, b), (P, k)
        assert np.array_equal(r[4], base[4][-(n // P):] if P > 1 else base[4]), P  # own kernel rows


def test_dshard_one_step_matches_oracle():
    n, dims, B = 8, [2, 64, 64, 1], 256
    x, y = synth.batch("gauss", B, 2, 1, 2)
    cfg = push.make_config(n, dims, max_batch=B, step_size=5e-2, seed=3, exchange="dshard")
    ctxs = push.local_group(cfg, 4)
    th = ctxs[0].gather("theta").astype(np.float64)
    for c in ctxs:
        c.particle_grads(_dev(x), _dev(y))
    for c in ctxs:
        c.svgd_step()
    G, _ = omlp.grads_all(th, dims, x, y)
    ref, _ = osvgd.svgd_step(th, G, 5e-2)
    assert rel_err(ctxs[2].gather("theta"), ref) <= 1e-4


def test_dshard_loopback_order_enforced():
    cfg = push.make_config(4, [1, 32, 1], max_batch=8, exchange="dshard")
    ctxs = push.local_group(cfg, 2)
    x = torch.zeros(8, 1, device="cuda")
    for c in ctxs:
        c.particle_grads(x, x)
    with pytest.raises(push.PushError) as e:
        ctxs[1].svgd_step()  # rank 0 has not called yet
    assert e.value.status == push.PUSH_E_STATE


SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from inputs import WORKLOADS, synth
from paper_2306_06528_b200 import push
w = WORKLOADS["C1"]
out = {{}}
for ex in ("allgather", "dshard"):
    for mode in ("eager", "graph"):
        ctx = push.Context(push.make_config(w.n_particles, list(w.dims), max_batch=w.batch, seed=3, step_size=1e-2,
                                            exchange=ex))
        for t in range(4):
            x, y = synth.workload_batch(w, t)
            xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
            if mode == "eager":
                ctx.particle_grads(xd, yd)
                ctx.svgd_step()
            else:
                ctx.step_graph(xd, yd)
        out[ex + mode] = (ctx.gather("theta"), ctx.gather("dist"))
np.savez({path!r}, **{{f"{{m}}_{{i}}": a for m, v in out.items() for i, a in enumerate(v)}})
"""


def test_dshard_nccl_send_recv_path_bit_identical(tmp_path):
    """PUSH_FORCE_NCCL=1: the transposes run as grouped ncclSend/ncclRecv (and the partials as an
    all-gather) on a single-rank communicator, eager and captured in the CUDA graph."""
    path = str(tmp_path / "ds.npz")
    env = dict(os.environ, PUSH_FORCE_NCCL="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, path=path)], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    a = np.load(path)
    for k in ("dshardeager", "dshardgraph", "allgathergraph"):
        for i in range(2):
            assert np.array_equal(a[f"{k}_{i}"], a[f"allgathereager_{i}"]), (k, i)
