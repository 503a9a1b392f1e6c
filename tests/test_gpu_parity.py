"""GPU path (libpush_b200.so through the C-ABI) vs the float64 oracle on the same seeded inputs.

Tolerances (north star / DESIGN.md §Parity):
  * g = grad log p:         ||g_gpu - g_ref||_inf / ||g_ref||_inf <= 1e-5 per particle (3xTF32)
  * one-step theta':        max rel err <= 1e-4 (floor 1e-3 * row max)
  * 100-step loss:          <= 1e-2 relative
  * init (K0), median bandwidth, sharding: bit-exact
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from inputs import WORKLOADS, synth  # noqa: E402
from oracle import init as oinit  # noqa: E402
from oracle import mlp as omlp  # noqa: E402
from oracle import svgd as osvgd  # noqa: E402
from paper_2306_06528_b200 import push  # noqa: E402

from .gpu_util import inf_rel, rel_err  # noqa: E402


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _d(dims):
    return sum(dims[l] * dims[l + 1] + dims[l + 1] for l in range(len(dims) - 1))


# ------------------------------------------------------------------ K0 init
@pytest.mark.parametrize("n,dims,seed", [(4, [1, 32, 32, 1], 0), (3, [2, 7, 5, 3], 11), (16, [2, 256, 256, 1], 5)])
def test_init_bit_exact(n, dims, seed):
    ctx = push.Context(push.make_config(n, dims, max_batch=8, seed=seed))
    th = ctx.gather("theta")
    assert np.array_equal(th, oinit.init_theta(n, dims, seed))


# ------------------------------------------------------------------ gradients a0-a5
GRAD_CASES = [
    # n, dims, B, act, prior, sigma, lam, data
    (4, [1, 32, 32, 1], 256, "tanh", "uniform", 1.0, 1.0, "sine"),        # C1 shape
    (3, [2, 64, 64, 64, 1], 300, "tanh", "uniform", 1.0, 1.0, "gauss"),   # ragged B
    (2, [3, 96, 32, 1], 128, "relu", "uniform", 1.0, 1.0, "gauss"),
    (3, [5, 7, 3], 50, "identity", "uniform", 1.0, 1.0, "gauss"),        # all thin layers
    (2, [32, 64, 1], 200, "tanh", "gaussian", 0.5, 2.0, "gauss"),         # layer 1 on tensor cores (X split)
    (2, [1, 33, 1], 64, "tanh", "uniform", 1.0, 1.0, "gauss"),            # width not % 32 -> thin path
    (2, [2, 128, 128, 1], 1, "tanh", "uniform", 1.0, 1.0, "gauss"),       # B = 1
    (2, [2, 256, 256, 256, 256, 1], 2048, "tanh", "uniform", 1.0, 1.0, "advection"),  # C2 net, split-K
    (3, [2, 64, 64, 33, 1], 200, "tanh", "uniform", 1.0, 1.0, "gauss"),   # GEMM layer under a thin hidden layer
    (2, [4, 64, 64, 2], 333, "tanh", "gaussian", 2.0, 1.0, "gauss"),      # d_out = 2, fused x0 with d_in = 4
    (2, [3, 128, 1], 8192, "tanh", "uniform", 1.0, 1.0, "burgers"),       # L = 2: output layer right above thin
    (2, [1, 33, 32, 32, 1], 160, "tanh", "uniform", 1.0, 1.0, "gauss"),   # GEMM layer with W not 16-B aligned
    # streaming output layer (output_stream_kernel): slab sizes, ragged blocks, d_out, activations
    (2, [4, 1], 100, "tanh", "uniform", 1.0, 1.0, "gauss"),               # L = 1: no delta below, shared x
    (2, [2, 64, 64, 3], 150, "identity", "uniform", 1.0, 1.0, "gauss"),   # d_out = 3 (DOUT 4), identity
    (2, [3, 1024, 1], 300, "tanh", "gaussian", 1.5, 1.0, "burgers"),     # 8-row slabs, 3-deep ring, ragged
    (2, [2, 2048, 1], 100, "tanh", "uniform", 1.0, 1.0, "gauss"),         # 4-row slabs, 8 features / thread
    (2, [2, 300, 2], 77, "relu", "uniform", 1.0, 1.0, "gauss"),           # H % 256 != 0, d_out = 2, relu
    # small ragged widths with relu + Gaussian prior; the C4 net shape
    (3, [2, 48, 40, 2], 130, "relu", "gaussian", 0.7, 1.5, "gauss"),
    (5, [1, 64, 64, 64, 1], 128, "tanh", "uniform", 1.0, 1.0, "random"),
]


@pytest.mark.parametrize("n,dims,B,act,prior,sigma,lam,data", GRAD_CASES)
def test_grads_match_oracle(n, dims, B, act, prior, sigma, lam, data):
    x, y = synth.batch(data, B, dims[0], dims[-1], step=3)
    cfg = push.make_config(n, dims, activation=act, prior=prior, prior_sigma=sigma, lik_scale=lam, max_batch=B + 7,
                           seed=2)
    ctx = push.Context(cfg)
    th = ctx.gather("theta")
    loss = torch.empty(n, device="cuda")
    ctx.particle_grads(_dev(x), _dev(y), loss)
    g = ctx.gather("grad")
    Gref, lref = omlp.grads_all(th, dims, x, y, act=act, lik_scale=lam, prior=prior, sigma=sigma)
    assert inf_rel(g, Gref) <= 1e-5
    np.testing.assert_allclose(loss.cpu().numpy(), lref, rtol=1e-5)
    np.testing.assert_allclose(ctx.gather("loss"), lref, rtol=1e-5)


# ------------------------------------------------------------------ kernel phase a7-a10
@pytest.mark.parametrize("n,d", [(1, 100), (2, 37), (3, 1000), (16, 5000), (33, 777), (64, 2048), (100, 96),
                                 (300, 64), (8, 70001), (4, 3333), (5, 4099), (6, 20000), (7, 131),
                                 # tensor-core update (n >= 128) with / without the Gram distances, ld padding
                                 (130, 999), (160, 3000), (96, 1537)])
def test_step_from_set_grads_matches_oracle(n, d):
    Th = synth.random_theta(n, d, seed=n + d, scale=0.2)
    G = synth.random_grads(n, d, seed=n * d)
    cfg = push.make_config(n, [d - 1, 1], max_batch=1, step_size=0.05)   # d = (d-1)*1 + 1 params
    assert _d(cfg_dims(cfg)) == d
    ctx = push.Context(cfg, theta0=Th)
    ctx.set_grads(_dev(G))
    ctx.svgd_step()
    th1 = ctx.gather("theta")
    ref, info = osvgd.svgd_step(Th, G, 0.05)
    assert rel_err(th1, ref) <= 1e-4
    D = ctx.gather("dist")
    assert np.array_equal(D, D.T) and np.all(np.diag(D) == 0)
    np.testing.assert_allclose(D, info["D"], rtol=1e-5, atol=1e-6 * max(info["D"].max(), 1e-30))
    h = float(ctx.gather("h")[0])
    assert h == pytest.approx(info["h"], rel=1e-5)
    K = ctx.gather("kernel")
    assert np.array_equal(K, K.T) and np.all(np.diag(K) == 1.0)


def cfg_dims(cfg):
    return [cfg.dims[i] for i in range(cfg.n_layers + 1)]


@pytest.mark.parametrize("n", [2, 3, 4, 9, 16, 25, 64, 128, 160, 256, 300])
def test_bandwidth_bit_exact_on_dyadic_lattice(n):
    """Dyadic Theta: every D_ij is exact in fp32 and fp64, so the GPU median equals the
    oracle's bit for bit and h = fp32(med) * fp32(1/ln n) (R4)."""
    d = 512
    Th = synth.dyadic_theta(n, d, seed=n)
    cfg = push.make_config(n, [d - 1, 1], max_batch=1)
    ctx = push.Context(cfg, theta0=Th)
    ctx.set_grads(_dev(np.zeros((n, d), np.float32)))
    ctx.svgd_step()
    D = ctx.gather("dist")
    Dref = osvgd.sq_dists(Th)
    assert np.array_equal(D.astype(np.float64), Dref)
    med = osvgd.median_all(Dref)
    expect = np.float32(med) * np.float32(1.0 / math.log(n))
    assert ctx.gather("h")[0] == expect


@pytest.mark.parametrize("rule", ["median_ln_n", "median_ln_n1", "fixed"])
@pytest.mark.parametrize("n", [5, 16, 64, 160, 256])
def test_bandwidth_reproduced_from_gpu_distances(rule, n):
    """Selection on the GPU's own fp32 D (oracle median, same precision) reproduces h bit-exactly."""
    d = 3000
    Th = synth.random_theta(n, d, seed=100 + n)
    cfg = push.make_config(n, [d - 1, 1], max_batch=1, bw_rule=rule, bw_h=0.75)
    ctx = push.Context(cfg, theta0=Th)
    ctx.set_grads(_dev(synth.random_grads(n, d, 3)))
    ctx.svgd_step()
    D = ctx.gather("dist")
    h = ctx.gather("h")[0]
    if rule == "fixed":
        assert h == np.float32(0.75)
        return
    med = np.float32(osvgd.median_all(D.astype(np.float64)))
    c = np.float32(1.0 / math.log(n if rule == "median_ln_n" else n + 1))
    assert h == med * c


@pytest.mark.parametrize("n,spread", [(16, 1e-2), (64, 1e-1), (64, 1e-2), (128, 1e-2), (256, 1e-3), (300, 1e-2)])
def test_clustered_particles_distances(n, spread):
    """theta_i = mu + spread * delta_i (|mu| ~ 1): the Gram form centred on particle 0 keeps D to the
    1e-5 bar where the uncentred Gram form cancels (R27), and the step matches."""
    d = 20000
    Th = synth.clustered_theta(n, d, seed=n, spread=spread)
    G = synth.random_grads(n, d, seed=5)
    ctx = push.Context(push.make_config(n, [d - 1, 1], max_batch=1, step_size=0.05), theta0=Th)
    ctx.set_grads(_dev(G))
    ctx.svgd_step()
    ref, info = osvgd.svgd_step(Th, G, 0.05)
    D = ctx.gather("dist")
    assert np.array_equal(D, D.T) and np.all(np.diag(D) == 0)
    off = ~np.eye(n, dtype=bool)
    assert np.max(np.abs(D[off] - info["D"][off]) / info["D"][off]) <= 1e-5
    assert float(ctx.gather("h")[0]) == pytest.approx(info["h"], rel=1e-5)
    assert rel_err(ctx.gather("theta"), ref) <= 1e-4


def test_single_particle_is_gradient_ascent():
    dims = [1, 32, 32, 1]
    x, y = synth.batch("sine", 256, 1, 1)
    ctx = push.Context(push.make_config(1, dims, max_batch=256, step_size=1e-2))
    th0 = ctx.gather("theta")
    ctx.particle_grads(_dev(x), _dev(y))
    ctx.svgd_step()
    assert ctx.gather("h")[0] == 1.0
    g, _ = omlp.grad_log_post(th0[0], dims, x, y)
    assert rel_err(ctx.gather("theta"), (th0[0] + 1e-2 * g)[None]) <= 1e-4


def test_coincident_particles_stay_coincident():
    d = 200
    th = np.tile(synth.random_theta(1, d, 1), (4, 1))
    G = np.tile(synth.random_grads(1, d, 2), (4, 1))
    ctx = push.Context(push.make_config(4, [d - 1, 1], max_batch=1), theta0=th)
    ctx.set_grads(_dev(G))
    ctx.svgd_step()
    t1 = ctx.gather("theta")
    assert ctx.gather("h")[0] == 1.0
    assert np.all(t1 == t1[0])


# ------------------------------------------------------------------ whole step, free running
def test_loss_trajectory_c1_100_steps():
    w = WORKLOADS["C1"]
    dims = list(w.dims)
    x, y = synth.workload_batch(w, 0)
    ctx = push.Context(push.make_config(w.n_particles, dims, max_batch=w.batch, step_size=1e-2, seed=0))
    th0 = ctx.gather("theta")
    xd, yd = _dev(x), _dev(y)
    losses = []
    loss = torch.empty(w.n_particles, device="cuda")
    for _ in range(100):
        ctx.particle_grads(xd, yd, loss)
        ctx.svgd_step()
        losses.append(loss.mean().item())
    _, ml, _, _ = osvgd.svgd_run(th0, dims, lambda t: (x, y), 100, 1e-2)
    np.testing.assert_allclose(np.array(losses), ml, rtol=1e-2)
    assert ml[-1] < ml[0]


@pytest.mark.parametrize("cfgname,steps", [("C2", 100), ("C4", 100), ("C5b", 5)])
def test_loss_trajectory_free_running(cfgname, steps):
    """Free-running loss trajectory (PAPER.md:661-664 loss tracking; north star: <= 1e-2 relative) of
    the bench path (push_step_graph after the eager first call) against the oracle's own run from the
    same K0 init and batches.  C5b (8 x 21M params) runs 5 steps: the fp64 oracle's update alone takes
    ~20 s per step there."""
    w = WORKLOADS[cfgname]
    dims = list(w.dims)
    ctx = push.Context(push.make_config(w.n_particles, dims, max_batch=w.batch, step_size=1e-3, seed=0))
    th0 = ctx.gather("theta")
    loss = torch.empty(w.n_particles, device="cuda")
    losses = []
    for t in range(steps):
        x, y = synth.workload_batch(w, t)
        ctx.step_graph(_dev(x), _dev(y), loss)
        losses.append(loss.double().mean().item())
    _, ml, _, _ = osvgd.svgd_run(th0, dims, lambda t: synth.workload_batch(w, t), steps, 1e-3)
    np.testing.assert_allclose(np.array(losses), ml, rtol=1e-2)


def test_step_host_equals_device_path():
    w = WORKLOADS["C1"]
    x, y = synth.workload_batch(w, 0)
    a = push.Context(push.make_config(w.n_particles, list(w.dims), max_batch=w.batch, seed=4))
    b = push.Context(push.make_config(w.n_particles, list(w.dims), max_batch=w.batch, seed=4))
    for _ in range(3):
        la = a.step_host(x, y)
        lb = torch.empty(w.n_particles, device="cuda")
        b.particle_grads(_dev(x), _dev(y), lb)
        b.svgd_step()
        assert np.array_equal(la, lb.cpu().numpy())
    assert np.array_equal(a.gather("theta"), b.gather("theta"))


# C4 / C5b: the captured step's side streams (a7-a9 beside the gradient phase; the loss reduction and
# weight gradients beside the backward GEMMs) over 3-6 hidden GEMM layers, the Gram form with the
# separate D kernel (n = 256) and the tensor-core update
@pytest.mark.parametrize("cfgname", ["C1", "C2", "C4", "C5b"])
def test_step_graph_equals_eager(cfgname):
    """push_step_graph (captured CUDA graph, batch staged into the context's buffers) reproduces the
    eager calls bit for bit over several steps with changing batches."""
    w = WORKLOADS[cfgname]
    dims = list(w.dims)
    a = push.Context(push.make_config(w.n_particles, dims, max_batch=w.batch, seed=6, step_size=1e-2))
    b = push.Context(push.make_config(w.n_particles, dims, max_batch=w.batch, seed=6, step_size=1e-2))
    la = torch.empty(w.n_particles, device="cuda")
    lb = torch.empty(w.n_particles, device="cuda")
    for t in range(5):
        x, y = synth.workload_batch(w, t)
        xd, yd = _dev(x), _dev(y)
        a.particle_grads(xd, yd, la)
        a.svgd_step()
        b.step_graph(xd, yd, lb)
        assert torch.equal(la, lb), t
    assert np.array_equal(a.gather("theta"), b.gather("theta"))
    assert np.array_equal(a.gather("dist"), b.gather("dist"))
    assert np.array_equal(a.gather("h"), b.gather("h"))
    assert np.array_equal(a.gather("kernel"), b.gather("kernel"))
    assert np.array_equal(a.gather("grad"), b.gather("grad"))


def test_step_graph_recapture_with_changing_batch():
    """Changing B between captured steps re-captures the graph (side streams, events, programmatic
    launches recorded afresh); every step stays bit-identical to the eager calls."""
    w = WORKLOADS["C2"]
    dims = list(w.dims)
    a = push.Context(push.make_config(w.n_particles, dims, max_batch=w.batch, seed=8, step_size=1e-2))
    b = push.Context(push.make_config(w.n_particles, dims, max_batch=w.batch, seed=8, step_size=1e-2))
    la = torch.empty(w.n_particles, device="cuda")
    lb = torch.empty(w.n_particles, device="cuda")
    for t, B in enumerate([w.batch, 1000, w.batch, 37, 37, w.batch]):
        x, y = synth.workload_batch(w, t)
        xd, yd = _dev(x[:B]), _dev(y[:B])
        a.particle_grads(xd, yd, la)
        a.svgd_step()
        b.step_graph(xd, yd, lb)
        assert torch.equal(la, lb), (t, B)
    assert np.array_equal(a.gather("theta"), b.gather("theta"))


def test_state_machine_errors():
    ctx = push.Context(push.make_config(2, [1, 32, 1], max_batch=8))
    with pytest.raises(push.PushError) as e:
        ctx.svgd_step()
    assert e.value.status == push.PUSH_E_STATE
    with pytest.raises(push.PushError) as e:
        ctx.gather("dist")
    assert e.value.status == push.PUSH_E_STATE
    x = torch.zeros(9, 1, device="cuda")
    with pytest.raises(push.PushError) as e:
        ctx.particle_grads(x, x)
    assert e.value.status == push.PUSH_E_SHAPE


# ------------------------------------------------------------------ sharding (loopback transport)
@pytest.mark.parametrize("dims,n,B", [([2, 64, 64, 1], 8, 256), ([1, 32, 32, 1], 4, 256),
                                      # n = 64: Gram-form distances; staged update at n_local = 64 / 32, the
                                      # 16-row kernel at n_local = 16 (same arithmetic)
                                      ([1, 32, 32, 1], 64, 128),
                                      # n = 128: Gram-form distances and the tensor-core update at every P
                                      ([1, 32, 32, 1], 128, 64)])
def test_sharding_bit_identical_across_P(dims, n, B):
    """Theta after 3 steps is bit-identical for P = 1, 2, 4 ranks."""
    x, y = synth.batch("gauss", B, dims[0], dims[-1], 1)
    xd, yd = _dev(x), _dev(y)
    results = {}
    for P in (1, 2, 4):
        if n % P:
            continue
        cfg = push.make_config(n, dims, max_batch=B, step_size=1e-2, seed=9)
        ctxs = push.local_group(cfg, P)
        for _ in range(3):
            for c in ctxs:
                c.particle_grads(xd, yd)
            for c in ctxs:
                c.svgd_step()
        results[P] = (ctxs[0].gather("theta"), ctxs[-1].gather("loss"), ctxs[0].gather("dist"))
    base = results[1]
    for P, r in results.items():
        assert np.array_equal(r[0], base[0]), P
        assert np.array_equal(r[1], base[1]), P
        assert np.array_equal(r[2], base[2]), P


# ------------------------------------------------------------------ 1-D Gaussian target through set_grads
def test_gaussian_target_closed_form_on_gpu():
    mu, sig, n = 1.0, 2.0, 64
    from scipy.stats import norm
    th = (mu + sig * norm.ppf((np.arange(n) + 0.5) / n)).reshape(n, 1).astype(np.float32)
    # dims [1, 1] -> d = 2 (w, b); the second coordinate is held at 0 with zero gradient
    theta0 = np.concatenate([th, np.zeros((n, 1), np.float32)], 1)
    ctx = push.Context(push.make_config(n, [1, 1], max_batch=1, step_size=0.2), theta0=theta0)
    for _ in range(800):
        t = torch.from_numpy(ctx.gather("theta")).cuda()
        g = -(t - mu) / sig ** 2
        g[:, 1] = 0.0
        ctx.set_grads(g.contiguous())
        ctx.svgd_step()
    t = ctx.gather("theta")[:, 0].astype(np.float64)
    assert abs(t.mean() - mu) < 1e-4
    assert abs(t.var() / sig ** 2 - 1.0) <= 0.08


# ------------------------------------------------------------------ full size (bench configuration, sampled)
def test_c2_full_size_sampled_parity():
    """BASELINE configs[1] at full size (16 x 198,401 params, B = 8192): g of sampled particles
    against the oracle one by one, and theta' of the whole step against the oracle's step."""
    w = WORKLOADS["C2"]
    dims = list(w.dims)
    x, y = synth.workload_batch(w, 0)
    ctx = push.Context(push.make_config(w.n_particles, dims, max_batch=w.batch, step_size=1e-3, seed=0))
    th0 = ctx.gather("theta")
    ctx.particle_grads(_dev(x), _dev(y))
    ctx.svgd_step()
    g = ctx.gather("grad")
    for i in (0, 7, 15):
        gref, _ = omlp.grad_log_post(th0[i], dims, x, y)
        assert inf_rel(g[i:i + 1], gref[None]) <= 1e-5, i
    ref, info = osvgd.svgd_step(th0, g.astype(np.float64), 1e-3)
    assert rel_err(ctx.gather("theta"), ref) <= 1e-4
    assert float(ctx.gather("h")[0]) == pytest.approx(info["h"], rel=1e-5)


@pytest.mark.parametrize("cfgname", ["S1", "C3", "C5"])
def test_full_size_sampled_parity_graph_path(cfgname):
    """Full-size configs through the bench's launch path — S1 (north-star point, 64 x 1,053,185 params,
    K = 512 GEMMs), C3 (64 x 3,153,921, K = 1024 GEMMs) and C5 (8 x 20,989,953, B = 1024, K = 2048 GEMMs)
    (push_step_graph after an eager warm-up step): g of sampled particles against the oracle one by one;
    D, h bit-compatible with the oracle's definition; theta' on sampled columns against the oracle's
    phi (column-separable) with the oracle's own K and h computed from the full Theta."""
    w = WORKLOADS[cfgname]
    dims = list(w.dims)
    ctx = push.Context(push.make_config(w.n_particles, dims, max_batch=w.batch, step_size=1e-3, seed=0))
    x0, y0 = synth.workload_batch(w, 0)
    ctx.step_graph(_dev(x0), _dev(y0))          # eager warm-up step (first call)
    x, y = synth.workload_batch(w, 1)
    th0 = ctx.gather("theta").astype(np.float64)
    ctx.step_graph(_dev(x), _dev(y))            # captured graph
    g = ctx.gather("grad")
    for i in (0, w.n_particles - 1):
        gref, _ = omlp.grad_log_post(th0[i], dims, x, y)
        assert inf_rel(g[i:i + 1], gref[None]) <= 1e-5, i
    D = osvgd.sq_dists(th0)
    h = osvgd.bandwidth(D)
    Dg = ctx.gather("dist").astype(np.float64)
    off = ~np.eye(w.n_particles, dtype=bool)
    assert np.max(np.abs(Dg[off] - D[off]) / D[off]) <= 1e-5
    assert float(ctx.gather("h")[0]) == pytest.approx(h, rel=1e-5)
    K = osvgd.kernel_matrix(D, h)
    rng = np.random.default_rng(0)
    cols = np.sort(rng.choice(th0.shape[1], 4096, replace=False))
    ref = th0[:, cols] + 1e-3 * osvgd.phi(th0[:, cols], g[:, cols].astype(np.float64), K, h)
    th1 = ctx.gather("theta")[:, cols]
    assert rel_err(th1, ref) <= 1e-4


# ------------------------------------------------------------------ predictive pushforward (NEXT-1)
@pytest.mark.parametrize("n,dims,B", [(4, [1, 32, 32, 1], 256), (16, [2, 256, 256, 256, 256, 1], 1000),
                                      (3, [5, 7, 3], 77), (8, [3, 96, 32, 2], 300)])
def test_predict_matches_oracle(n, dims, B):
    from oracle import predict as opred
    x, _ = synth.batch("gauss", B, dims[0], dims[-1], step=5)
    ctx = push.Context(push.make_config(n, dims, max_batch=B, seed=4))
    th = ctx.gather("theta")
    pred, mean, std = ctx.predict(_dev(x))
    rp, rm, rs = opred.predictive_summary(th, dims, x)
    assert inf_rel(pred.cpu().numpy().reshape(n, -1), rp.reshape(n, -1)) <= 1e-5
    scale = np.abs(rp).max()
    np.testing.assert_allclose(mean.cpu().numpy(), rm, rtol=0, atol=1e-5 * scale)
    np.testing.assert_allclose(std.cpu().numpy(), rs, rtol=0, atol=1e-5 * scale)
    # the training state is untouched: a step after predict equals a step without it
    x2, y2 = synth.batch("gauss", B, dims[0], dims[-1], step=6)
    ctx2 = push.Context(push.make_config(n, dims, max_batch=B, seed=4))
    for c in (ctx, ctx2):
        c.particle_grads(_dev(x2), _dev(y2))
        c.svgd_step()
    assert np.array_equal(ctx.gather("theta"), ctx2.gather("theta"))


# ------------------------------------------------------------------ NEXT-3: deep ensembles, diagonal SWAG
def test_ensemble_step_and_swag_match_oracle():
    from oracle import swag as oswag
    w = WORKLOADS["C1"]
    dims = list(w.dims)
    x, y = synth.workload_batch(w, 0)
    ctx = push.Context(push.make_config(w.n_particles, dims, max_batch=w.batch, step_size=5e-2, seed=8, swag=True))
    snaps = []
    for t in range(4):
        th = ctx.gather("theta")
        ctx.particle_grads(_dev(x), _dev(y))
        ctx.ensemble_step()
        g = ctx.gather("grad")
        assert rel_err(ctx.gather("theta"), oswag.ensemble_step(th, g, 5e-2)) <= 1e-6
        ctx.swag_collect()
        snaps.append(ctx.gather("theta"))
    mean, mom2, _ = oswag.swag_moments(snaps)
    z = oswag.swag_normal(99, 0, w.n_particles, ctx.d)
    ref = oswag.swag_sample(mean, mom2, z)
    smp = ctx.swag_sample(99).cpu().numpy()
    sd = np.sqrt(np.maximum(mom2 - mean * mean, 0.0))
    # fp32 moments: mom2 - mean^2 cancels, so the variance is only known to ~fp32 eps * (mom2 + mean^2);
    # elementwise bound: |z| sqrt(that) + 1e-5 (|mean| + |z| sd)
    var_err = 4.0 * np.finfo(np.float32).eps * (mom2 + mean * mean)
    tol = np.abs(z) * np.sqrt(var_err) + 1e-5 * (np.abs(mean) + np.abs(z) * sd) + 1e-7
    assert np.all(np.abs(smp - ref) <= tol)
    assert np.array_equal(smp, ctx.swag_sample(99).cpu().numpy())      # same seed, same draw
    with pytest.raises(push.PushError):
        push.Context(push.make_config(2, [1, 4, 1], max_batch=4)).swag_collect()   # cfg.swag = 0
