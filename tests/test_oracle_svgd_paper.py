"""Pins for oracle.svgd_paper — PusH's own update:
closed forms, reductions to the pinned canonical step, a finite-difference check of the repulsion
and invariances that a wrong tensor split, weight or sign would break."""
import math

import numpy as np
import pytest

from oracle import mlp, svgd, svgd_paper

DIMS = [2, 3, 4, 1]  # tensors: W0 3x2, b0 3, W1 4x3, b1 4, W2 1x4, b2 1  -> d = 6+3+12+4+4+1 = 30


def _setup(n, seed, dims=DIMS, s=0.4):
    rng = np.random.default_rng(seed)
    d = sum(dims[l] * dims[l + 1] + dims[l + 1] for l in range(len(dims) - 1))
    return rng.standard_normal((n, d)) * s, rng.standard_normal((n, d)), d


def test_tensor_ranges_follow_parameter_order():
    r = svgd_paper.tensor_ranges(DIMS)
    assert r == [(0, 6), (6, 3), (9, 12), (21, 4), (25, 4), (29, 1)]
    # the same blocks as the oracle's own unpacking of the canonical layout (R15)
    theta = np.arange(30.0)
    layers = mlp.unpack(theta, DIMS)
    flat = []
    for W, b in layers:
        flat += [W.ravel(), b.ravel()]
    for (off, size), blk in zip(r, flat):
        assert np.array_equal(theta[off:off + size], blk)


@pytest.mark.parametrize("rule", [svgd.BW_MEDIAN_LN_N, svgd.BW_FIXED])
def test_all_switches_off_is_the_canonical_step(rule):
    Th, G, _ = _setup(6, 1)
    a, ia = svgd_paper.svgd_step_variant(Th, G, 0.05, DIMS, per_tensor=False, paper_norm=False, prior_sum=False,
                                         rule=rule, h_fixed=1.3)
    b, ib = svgd.svgd_step(Th, G, 0.05, rule, 1.3)
    np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-15)
    assert ia["h"][0] == pytest.approx(ib["h"], rel=1e-15)


@pytest.mark.parametrize("paper_norm", [False, True])
@pytest.mark.parametrize("prior_sum", [False, True])
def test_two_particles_closed_form(paper_norm, prior_sum):
    # n = 2, per tensor t with k_t = exp(-|d_t|^2 / h):  phi_1 = w(g_1 + k_t g_2) + (1/2)(2/h) k_t (th_1 - th_2)
    #                                                               [+ w (p0'(th_1) + p0'(th_2))]
    Th, G, d = _setup(2, 2)
    sigma, eps, h = 0.7, 0.1, 2.0
    new, _ = svgd_paper.svgd_step_variant(Th, G, eps, DIMS, True, paper_norm, prior_sum, prior="gaussian",
                                          sigma=sigma, rule=svgd.BW_FIXED, h_fixed=h)
    w = 1.0 if paper_norm else 0.5
    for off, size in svgd_paper.tensor_ranges(DIMS):
        a, b = Th[0, off:off + size], Th[1, off:off + size]
        k = math.exp(-float(((a - b) ** 2).sum()) / h)
        phi1 = w * (G[0, off:off + size] + k * G[1, off:off + size]) + 0.5 * (2.0 / h) * k * (a - b)
        phi2 = w * (G[1, off:off + size] + k * G[0, off:off + size]) + 0.5 * (2.0 / h) * k * (b - a)
        if prior_sum:
            pr = -(a + b) / sigma ** 2
            phi1, phi2 = phi1 + w * pr, phi2 + w * pr
        np.testing.assert_allclose(new[0, off:off + size], a + eps * phi1, rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(new[1, off:off + size], b + eps * phi2, rtol=1e-13, atol=1e-15)


def test_repulsion_is_minus_gradient_of_total_tensor_similarity():
    # G = 0, paper normalisation: (theta_i' - theta_i)/eps = -(1/n) grad_{theta_i} sum_t sum_j k_t(theta_j, theta_i)
    n, h, eps = 5, 1.7, 1.0
    Th, _, d = _setup(n, 3)
    new, _ = svgd_paper.svgd_step_variant(Th, np.zeros_like(Th), eps, DIMS, True, True, False,
                                          rule=svgd.BW_FIXED, h_fixed=h)
    ranges = svgd_paper.tensor_ranges(DIMS)

    def f(x, i):
        tot = 0.0
        for j in range(n):
            for off, size in ranges:
                tot += math.exp(-float(((x[off:off + size] - Th[j, off:off + size]) ** 2).sum()) / h)
        return tot

    i, step = 2, 1e-6
    fd = np.empty(d)
    for k in range(d):
        e = np.zeros(d)
        e[k] = step
        fd[k] = (f(Th[i] + e, i) - f(Th[i] - e, i)) / (2 * step)
    np.testing.assert_allclose((new[i] - Th[i]) / eps, -fd / n, rtol=1e-6, atol=1e-9)


def test_one_differing_tensor_matches_the_whole_theta_kernel():
    # every tensor but W1 identical across particles: W1's columns see the whole-theta kernel, the
    # others K = 1 (no repulsion, drive = mean of g)
    n = 6
    Th, G, d = _setup(n, 4)
    off, size = svgd_paper.tensor_ranges(DIMS)[2]
    mask = np.zeros(d, bool)
    mask[off:off + size] = True
    Th[:, ~mask] = Th[0, ~mask]
    a, info = svgd_paper.svgd_step_variant(Th, G, 0.05, DIMS, True, False, False, rule=svgd.BW_MEDIAN_LN_N)
    b, ib = svgd.svgd_step(Th, G, 0.05, svgd.BW_MEDIAN_LN_N)
    np.testing.assert_allclose(a[:, mask], b[:, mask], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(a[:, ~mask], Th[:, ~mask] + 0.05 * G[:, ~mask].mean(0), rtol=1e-12, atol=1e-15)
    assert info["h"][2] == pytest.approx(ib["h"], rel=1e-14)
    assert all(h == 1.0 for t, h in enumerate(info["h"]) if t != 2)  # median 0 -> h = 1 (R4)


def test_per_tensor_median_bandwidth_is_scale_covariant_per_tensor():
    # scaling one tensor by c scales only its h by c^2 and leaves every K_t unchanged
    n, c = 7, 3.0
    Th, G, _ = _setup(n, 5)
    off, size = svgd_paper.tensor_ranges(DIMS)[4]
    Th2 = Th.copy()
    Th2[:, off:off + size] *= c
    _, i1 = svgd_paper.svgd_step_variant(Th, G, 0.01, DIMS, True, True, False, rule=svgd.BW_MEDIAN_LN_N)
    _, i2 = svgd_paper.svgd_step_variant(Th2, G, 0.01, DIMS, True, True, False, rule=svgd.BW_MEDIAN_LN_N)
    for t in range(len(i1["h"])):
        assert i2["h"][t] == pytest.approx(i1["h"][t] * (c * c if t == 4 else 1.0), rel=1e-12)
    np.testing.assert_allclose(i1["K"], i2["K"], rtol=1e-12)


@pytest.mark.parametrize("paper_norm", [False, True])
def test_unweighted_prior_equals_weighted_when_particles_coincide(paper_norm):
    # all particles equal -> every K = 1, so sum_j w p0'(theta_j) equals sum_j w K_ij p0'(theta_j)
    n, sigma = 5, 0.9
    Th, G, _ = _setup(n, 6)
    Th[:] = Th[0]
    a, _ = svgd_paper.svgd_step_variant(Th, G, 0.02, DIMS, True, paper_norm, True, prior="gaussian", sigma=sigma)
    Gfull = G + mlp.prior_grad(Th[0], "gaussian", sigma)
    b, _ = svgd_paper.svgd_step_variant(Th, Gfull, 0.02, DIMS, True, paper_norm, False)
    np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-15)


def test_paper_norm_scales_drive_by_n_only():
    # with h huge, K ~ 1 and the repulsion ~ 0: paper_norm's drive is n times the canonical one
    n = 4
    Th, G, _ = _setup(n, 7)
    a, _ = svgd_paper.svgd_step_variant(Th, G, 1.0, DIMS, False, True, False, rule=svgd.BW_FIXED, h_fixed=1e12)
    b, _ = svgd_paper.svgd_step_variant(Th, G, 1.0, DIMS, False, False, False, rule=svgd.BW_FIXED, h_fixed=1e12)
    np.testing.assert_allclose(a - Th, n * (b - Th), rtol=1e-9)
