"""Pins for oracle.svgd: what the paper and the mathematics of SVGD fix
(north star list; SURVEY.md §8(c) 'What pins each part')."""
import math

import numpy as np
import pytest
from scipy.stats import norm

from oracle import mlp, svgd


def _rand(n, d, seed, s=0.3):
    return np.random.default_rng(seed).standard_normal((n, d)) * s


# ---------------------------------------------------------------- distances / kernel
def test_distances_and_kernel_symmetric_unit_diagonal():
    Th = _rand(7, 13, 0)
    D = svgd.sq_dists(Th)
    assert np.array_equal(D, D.T) and np.all(np.diag(D) == 0.0)
    # brute force definition on one pair
    assert D[2, 5] == pytest.approx(sum((Th[2, k] - Th[5, k]) ** 2 for k in range(13)), rel=1e-14)
    K = svgd.kernel_matrix(D, 0.7)
    assert np.array_equal(K, K.T) and np.all(np.diag(K) == 1.0)
    assert np.all((K > 0) & (K <= 1))


def test_kernel_worked_example():
    # ||a-b||^2 = 2 with h = 2 -> e^{-1}  (SPEC.md:103 under R1)
    Th = np.array([[0.0, 0.0], [1.0, 1.0]])
    D = svgd.sq_dists(Th)
    assert D[0, 1] == 2.0
    assert svgd.kernel_matrix(D, 2.0)[0, 1] == pytest.approx(math.exp(-1.0), rel=1e-15)


# ---------------------------------------------------------------- median / bandwidth
@pytest.mark.parametrize("n", range(1, 13))
def test_median_matches_brute_force_and_triangle_rank_map(n):
    Th = _rand(n, 5, 10 + n)
    D = svgd.sq_dists(Th)
    vals = sorted(D[i, j] for i in range(n) for j in range(n))
    N = n * n
    brute = vals[N // 2] if N % 2 else 0.5 * (vals[N // 2 - 1] + vals[N // 2])
    assert svgd.median_all(D) == brute
    # SURVEY.md §8(c) step 3 closed-form mapping onto the strict upper triangle
    u = sorted(D[i, j] for i in range(n) for j in range(i + 1, n))
    if n == 1:
        m = 0.0
    elif n == 2:
        m = u[0] / 2
    elif n % 2 == 0:
        r = n * (n - 2) // 4
        m = (u[r - 1] + u[r]) / 2
    else:
        m = u[(n - 1) ** 2 // 4 - 1]
    assert svgd.median_all(D) == pytest.approx(m, rel=1e-15)


def test_bandwidth_rules_and_degenerate_cases():
    D = svgd.sq_dists(_rand(5, 3, 1))
    med = float(np.median(D))
    assert svgd.bandwidth(D, svgd.BW_MEDIAN_LN_N) == pytest.approx(med / math.log(5))
    assert svgd.bandwidth(D, svgd.BW_MEDIAN_LN_N1) == pytest.approx(med / math.log(6))
    assert svgd.bandwidth(D, svgd.BW_FIXED, 2.5) == 2.5
    assert svgd.bandwidth(np.zeros((1, 1))) == 1.0                     # n = 1
    assert svgd.bandwidth(svgd.sq_dists(np.ones((4, 3)))) == 1.0        # med = 0


def test_median_rule_closed_forms():
    """Under MEDIAN_LN_N, K_ij = n^(-D_ij/med): n=2 -> K_12 = 1/4; n=3 closest pair -> 1/3;
    odd n: a median-distance pair has K = 1/n; MEDIAN_LN_N1 at n=2 -> 1/9."""
    Th2 = _rand(2, 6, 2)
    D = svgd.sq_dists(Th2)
    assert svgd.kernel_matrix(D, svgd.bandwidth(D))[0, 1] == pytest.approx(0.25, rel=1e-14)
    assert svgd.kernel_matrix(D, svgd.bandwidth(D, svgd.BW_MEDIAN_LN_N1))[0, 1] == pytest.approx(1 / 9, rel=1e-14)
    Th3 = _rand(3, 4, 3)
    D3 = svgd.sq_dists(Th3)
    K3 = svgd.kernel_matrix(D3, svgd.bandwidth(D3))
    iu = np.triu_indices(3, 1)
    assert K3[iu].max() == pytest.approx(1 / 3, rel=1e-13)
    for n in (5, 7, 9):
        Dn = svgd.sq_dists(_rand(n, 3, 40 + n))
        Kn = svgd.kernel_matrix(Dn, svgd.bandwidth(Dn))
        med = float(np.median(Dn))
        i, j = np.argwhere(Dn == med)[0]
        assert Kn[i, j] == pytest.approx(1.0 / n, rel=1e-13)


def test_two_particle_step_closed_form():
    # phi_1 = 1/2 [g_1 + g_2/4 + (ln2/D_12)(theta_1 - theta_2)]  (2/h = 4 ln2 / D_12, K_12 = 1/4)
    Th = _rand(2, 5, 5)
    G = _rand(2, 5, 6, 1.0)
    _, info = svgd.svgd_step(Th, G, 1e-3)
    D12 = float(np.sum((Th[0] - Th[1]) ** 2))
    expect = 0.5 * (G[0] + G[1] / 4 + (math.log(2) / D12) * (Th[0] - Th[1]))
    assert np.allclose(info["phi"][0], expect, rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- repulsion
def test_repulsion_is_minus_grad_of_kernel_row_sum():
    """sum_j grad_{theta_j} K_ij = -grad_{theta_i} sum_j K_ij (h frozen), by central differences."""
    n, d, h = 4, 6, 0.8
    Th = _rand(n, d, 7)
    K = svgd.kernel_matrix(svgd.sq_dists(Th), h)
    rep = svgd.phi(Th, np.zeros_like(Th), K, h) * n   # G = 0 isolates the repulsive sum
    for i in range(n):
        def rowsum(ti):
            T = Th.copy(); T[i] = ti
            return svgd.kernel_matrix(svgd.sq_dists(T), h)[i].sum()
        for k in range(d):
            e = np.zeros(d); e[k] = 1e-6
            fd = (rowsum(Th[i] + e) - rowsum(Th[i] - e)) / 2e-6
            assert -fd == pytest.approx(rep[i, k], rel=1e-6, abs=1e-9)


# ---------------------------------------------------------------- whole-step special cases
def test_single_particle_is_gradient_ascent():
    """n = 1: phi = g exactly, so 100 SVGD steps == 100 steps of theta += eps g."""
    dims = (1, 6, 6, 1)
    d = 1 * 6 + 6 + 36 + 6 + 6 + 1
    th = _rand(1, d, 8, 0.5)
    x = np.linspace(-1, 1, 32).reshape(32, 1); y = np.sin(3 * x)
    A = th.copy(); Bv = th[0].copy()
    for _ in range(100):
        G, _ = mlp.grads_all(A, dims, x, y)
        A, info = svgd.svgd_step(A, G, 1e-2)
        assert info["h"] == 1.0
        g, _ = mlp.grad_log_post(Bv, dims, x, y)
        Bv = Bv + 1e-2 * g
    assert np.array_equal(A[0], Bv)


def test_three_particle_brute_force_double_loop():
    """n = 3, a 2-parameter model: phi against a scalar triple loop of the definition."""
    Th = _rand(3, 2, 9)
    G = _rand(3, 2, 10, 1.0)
    h = 0.9
    K = svgd.kernel_matrix(svgd.sq_dists(Th), h)
    ph = svgd.phi(Th, G, K, h)
    for i in range(3):
        for k in range(2):
            s = 0.0
            for j in range(3):
                r2 = (Th[i, 0] - Th[j, 0]) ** 2 + (Th[i, 1] - Th[j, 1]) ** 2
                kij = math.exp(-r2 / h)
                s += kij * G[j, k] + kij * 2.0 / h * (Th[i, k] - Th[j, k])
            assert ph[i, k] == pytest.approx(s / 3, rel=1e-12, abs=1e-14)


def test_flat_kernel_preserves_differences():
    """h -> infinity with a shared gradient: K -> 1, repulsion -> 0; pairwise differences kept."""
    Th = _rand(5, 8, 11)
    G = np.tile(_rand(1, 8, 12, 1.0), (5, 1))
    new, _ = svgd.svgd_step(Th, G, 1e-2, svgd.BW_FIXED, 1e12)
    diff0 = Th[:, None, :] - Th[None, :, :]
    diff1 = new[:, None, :] - new[None, :, :]
    assert np.max(np.abs(diff1 - diff0)) < 1e-8


def test_coincident_particles_and_fixed_point():
    th = _rand(1, 7, 13)
    Th = np.tile(th, (4, 1))
    G = np.tile(_rand(1, 7, 14, 1.0), (4, 1))
    new, info = svgd.svgd_step(Th, G, 1e-2)
    assert info["h"] == 1.0                      # med = 0 -> h = 1 (R4)
    assert np.all(new == new[0])                 # coincident particles stay coincident
    new0, info0 = svgd.svgd_step(Th, np.zeros_like(Th), 1e-2)
    assert np.all(info0["phi"] == 0.0) and np.array_equal(new0, Th)   # fixed point


def test_translation_and_permutation_equivariance():
    Th = _rand(6, 9, 15)
    G = _rand(6, 9, 16, 1.0)
    c = _rand(1, 9, 17, 3.0)
    a, _ = svgd.svgd_step(Th, G, 1e-2)
    b, _ = svgd.svgd_step(Th + c, G, 1e-2)
    assert np.allclose(b, a + c, rtol=0, atol=1e-12)
    p = np.random.default_rng(18).permutation(6)
    e, _ = svgd.svgd_step(Th[p], G[p], 1e-2)
    assert np.allclose(e, a[p], rtol=1e-13, atol=1e-15)


def test_gaussian_target_closed_form_mean_and_variance():
    """1-D target N(mu, sigma^2), g = -(x - mu)/sigma^2: a symmetric init keeps mean = mu
    (to 1e-12, exact by symmetry); variance reaches the finite-n SVGD fixed point
    (var/sigma^2 = 0.946 at n = 64) -> |var/sigma^2 - 1| <= 0.08."""
    mu, sig, n = 1.0, 2.0, 64
    Th = (mu + sig * norm.ppf((np.arange(n) + 0.5) / n)).reshape(n, 1)
    for _ in range(800):
        Th, _ = svgd.svgd_step(Th, -(Th - mu) / sig ** 2, 0.2)
    assert abs(Th.mean() - mu) < 1e-12
    assert abs(Th.var() / sig ** 2 - 1.0) <= 0.08
    assert Th.var() < sig ** 2          # known finite-n bias is below sigma^2


def test_run_records_pre_update_losses():
    dims = (1, 4, 1)
    Th0 = _rand(3, 1 * 4 + 4 + 4 + 1, 19, 0.5)
    x = np.linspace(-1, 1, 8).reshape(8, 1); y = np.sin(x)
    ThT, ml, l0, hs = svgd.svgd_run(Th0, dims, lambda t: (x, y), 3, 1e-2)
    _, losses = mlp.grads_all(Th0, dims, x, y)
    assert ml[0] == pytest.approx(losses.mean()) and l0[0] == pytest.approx(losses[0])
    assert len(hs) == 3 and ThT.shape == Th0.shape
