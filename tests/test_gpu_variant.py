"""NEXT-2 on the GPU: PusH's own update (push_config.variant, include/push.h PUSH_VAR_*) through the
C-ABI vs oracle.svgd_paper on the same seeded inputs.

Tolerances as the canonical step (tests/test_gpu_parity.py): theta' max rel err <= 1e-4, distances
1e-5 relative, per-tensor median bandwidth 1e-5; graph == eager and P = 1/2/4 sharding bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import synth  # noqa: E402
from oracle import mlp as omlp  # noqa: E402
from oracle import svgd as osvgd  # noqa: E402
from oracle import svgd_paper as opaper  # noqa: E402
from paper_2306_06528_b200 import push  # noqa: E402

from .gpu_util import inf_rel, rel_err  # noqa: E402

RULE = {"fixed": osvgd.BW_FIXED, "median": osvgd.BW_MEDIAN_LN_N, "median_ln_n1": osvgd.BW_MEDIAN_LN_N1}


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _d(dims):
    return sum(dims[l] * dims[l + 1] + dims[l + 1] for l in range(len(dims) - 1))


def _flags(v):
    return dict(per_tensor=bool(v & push.VAR_PER_TENSOR), paper_norm=bool(v & push.VAR_PAPER_NORM),
                prior_sum=bool(v & push.VAR_PRIOR_SUM))


CASES = [
    # n, dims, variant, bw rule
    (5, [3, 5, 7, 2], 7, "fixed"),          # odd tensor sizes: every split range unaligned
    (5, [3, 5, 7, 2], 1, "median"),
    (1, [3, 5, 7, 2], 7, "median"),         # n = 1
    (40, [1, 33, 32, 1], 7, "median"),      # several row tiles, ragged rows, 33-wide tensors
    (40, [1, 33, 32, 1], 2, "median_ln_n1"),
    (16, [2, 256, 256, 1], 7, "fixed"),     # a 65,536-element tensor over several splits (C2-like widths)
    (16, [2, 256, 256, 1], 3, "median"),
    (9, [4, 64, 64, 2], 4, "median"),       # prior sum alone, whole-theta kernel
    (9, [4, 64, 64, 2], 5, "fixed"),
    (9, [4, 64, 64, 2], 6, "median"),
    (20, [2, 16, 1], 7, "median"),          # d_out = 1 bias: a 1-element tensor
]


@pytest.mark.parametrize("n,dims,variant,rule", CASES)
def test_variant_step_from_set_grads_matches_oracle(n, dims, variant, rule):
    d = _d(dims)
    Th = synth.random_theta(n, d, seed=n + d + variant, scale=0.25)
    G = synth.random_grads(n, d, seed=3 * n + variant)
    sigma, eps, h_fixed = 0.8, 0.02, 2.0
    cfg = push.make_config(n, dims, max_batch=1, step_size=eps, prior="gaussian", prior_sigma=sigma, bw_rule=rule,
                           bw_h=h_fixed, variant=variant)
    ctx = push.Context(cfg, theta0=Th)
    ctx.set_grads(_dev(G))
    ctx.svgd_step()
    th1 = ctx.gather("theta")
    ref, info = opaper.svgd_step_variant(Th, G, eps, dims, prior="gaussian", sigma=sigma, rule=RULE[rule],
                                         h_fixed=h_fixed, **_flags(variant))
    assert rel_err(th1, ref) <= 1e-4
    T = len(info["ranges"])
    D = ctx.gather("dist").reshape(T, n, n)
    for t in range(T):
        Dt = D[t]
        assert np.array_equal(Dt, Dt.T) and np.all(np.diag(Dt) == 0)
        np.testing.assert_allclose(Dt, info["D"][t], rtol=1e-5, atol=1e-6 * max(info["D"][t].max(), 1e-30))
    np.testing.assert_allclose(ctx.gather("h"), info["h"], rtol=1e-5)
    K = ctx.gather("kernel").reshape(T, n, n)
    assert np.all(K[:, np.arange(n), np.arange(n)] == 1.0)


def test_variant_paper_full_path_matches_oracle():
    """Gradients (likelihood term only under PRIOR_SUM) + PusH's update, 3 steps on a C1-shaped net
    with a Gaussian prior, against the oracle's mlp + svgd_paper."""
    n, dims, B, sigma, eps = 4, [1, 32, 32, 1], 256, 1.5, 1e-2
    cfg = push.make_config(n, dims, max_batch=B, step_size=eps, prior="gaussian", prior_sigma=sigma, bw_rule="fixed",
                           bw_h=2.0, seed=5, variant=push.VARIANT_PAPER)
    ctx = push.Context(cfg)
    Th = ctx.gather("theta").astype(np.float64)
    for t in range(3):
        x, y = synth.batch("sine", B, 1, 1, t)
        ctx.particle_grads(_dev(x), _dev(y))
        G, _ = omlp.grads_all(Th, dims, x, y, prior="uniform")
        assert inf_rel(ctx.gather("grad"), G) <= 1e-5  # the prior is not in G under PRIOR_SUM
        ctx.svgd_step()
        Th, _ = opaper.svgd_step_variant(Th, G, eps, dims, prior="gaussian", sigma=sigma, rule=osvgd.BW_FIXED,
                                         h_fixed=2.0)
        assert rel_err(ctx.gather("theta"), Th) <= 1e-4, t
        Th = ctx.gather("theta").astype(np.float64)  # continue from the GPU state (one-step parity each step)


def test_variant_graph_equals_eager_and_sharding_bit_exact():
    n, dims, B = 8, [2, 64, 64, 1], 256
    x, y = synth.batch("gauss", B, 2, 1, 1)
    xd, yd = _dev(x), _dev(y)
    mk = lambda: push.make_config(n, dims, max_batch=B, step_size=1e-2, seed=9, prior="gaussian", prior_sigma=1.0,
                                  bw_rule="median", variant=push.VARIANT_PAPER)
    a, b = push.Context(mk()), push.Context(mk())
    for _ in range(3):
        a.particle_grads(xd, yd)
        a.svgd_step()
        b.step_graph(xd, yd)
    assert np.array_equal(a.gather("theta"), b.gather("theta"))
    base = a.gather("theta")
    for P in (2, 4):
        ctxs = push.local_group(mk(), P)
        for _ in range(3):
            for c in ctxs:
                c.particle_grads(xd, yd)
            for c in ctxs:
                c.svgd_step()
        assert np.array_equal(ctxs[0].gather("theta"), base), P
        assert np.array_equal(ctxs[0].gather("dist"), a.gather("dist")), P


def test_canonical_path_unchanged_by_the_split_table():
    """variant = 0 keeps the canonical whole-row plan: same D as the oracle's and T = 1 shapes."""
    n, d = 33, 777
    Th = synth.random_theta(n, d, seed=1, scale=0.2)
    G = synth.random_grads(n, d, seed=2)
    ctx = push.Context(push.make_config(n, [d - 1, 1], max_batch=1, step_size=0.05), theta0=Th)
    ctx.set_grads(_dev(G))
    ctx.svgd_step()
    ref, info = osvgd.svgd_step(Th, G, 0.05)
    assert ctx.gather("dist").shape == (n, n) and ctx.gather("h").shape == (1,)
    assert rel_err(ctx.gather("theta"), ref) <= 1e-4
