"""ORACLE (test infrastructure) — the SVGD particle step of PusH in float64.

Passages followed
-----------------
* SVGD direction (north star; "performs the SVGD update by
  computing a step using a pairwise comparison using the kernel w.r.t. every
  other particle"; code PAPER.md:612-641, Fig. supp:svgd):

      phi(theta_i) = (1/n) sum_j [ K_ij grad log p(theta_j) + grad_{theta_j} K_ij ]

  with the RBF kernel K_ij = exp(-||theta_i - theta_j||^2 / h) over the whole
  flattened theta (R1, R6), hence grad_{theta_j} K_ij = (2/h)(theta_i - theta_j) K_ij.
  j runs over all n particles, j = i included (R11).
* Bandwidth: median heuristic of the SVGD paper the PusH paper builds on
  (PAPER.md:24/71 cite liuSteinVariationalGradient2016): h = med / ln n with
  med the median of all n^2 squared distances (R3, R4); FIXED h for the paper's
  own "kernel_bandwidth" (R2).
* Step: theta_i <- theta_i + eps * phi(theta_i) for every i simultaneously
  (Jacobi, R10; sign convention R7: ascent on log p).
* Gradients g_j come from oracle.mlp or are supplied.

The update below is written as the paper's double loop over (i, j) (vectorised
only over the parameter axis), not in the fused form the GPU uses.
Pins: tests/test_oracle_svgd.py.
"""
from __future__ import annotations

import math

import numpy as np

from . import mlp

BW_MEDIAN_LN_N = 0
BW_MEDIAN_LN_N1 = 1
BW_FIXED = 2


def sq_dists(Theta):
    """D_ij = sum_k (theta_ik - theta_jk)^2 for all i, j (exactly symmetric, zero diagonal)."""
    Theta = np.asarray(Theta, dtype=np.float64)
    n = Theta.shape[0]
    D = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1, n):          # (a-b)^2 == (b-a)^2 exactly: fill both triangles
            diff = Theta[i] - Theta[j]
            D[i, j] = D[j, i] = float(np.dot(diff, diff))
    return D


def median_all(D):
    """numpy median of all n^2 entries (average of the two middle order statistics if n^2 even; R3)."""
    return float(np.median(np.asarray(D, dtype=np.float64).ravel()))


def bandwidth(D, rule=BW_MEDIAN_LN_N, h_fixed=1.0):
    """h per R2-R4: median/ln n (default), median/ln(n+1), or fixed; h = 1 if n = 1 or med <= 0."""
    n = D.shape[0]
    if rule == BW_FIXED:
        return float(h_fixed)
    med = median_all(D)
    if n == 1 or med <= 0.0:
        return 1.0
    denom = math.log(n) if rule == BW_MEDIAN_LN_N else math.log(n + 1)
    return med / denom


def kernel_matrix(D, h):
    """K_ij = exp(-D_ij / h)  (RBF over the flattened theta, R1/R6)."""
    return np.exp(-np.asarray(D, dtype=np.float64) / h)


def phi(Theta, G, K, h):
    """phi(theta_i) = (1/n) sum_j [K_ij g_j + grad_{theta_j} K_ij],
    grad_{theta_j} K_ij = (2/h)(theta_i - theta_j) K_ij   (north star)."""
    Theta = np.asarray(Theta, dtype=np.float64)
    G = np.asarray(G, dtype=np.float64)
    n = Theta.shape[0]
    K = np.asarray(K, dtype=np.float64)
    acc = np.zeros_like(Theta)                  # row i accumulates particle i's sum over j
    for j in range(n):
        kj = K[:, j:j + 1]                      # K_ij for every i
        acc += kj * G[j]                        # attractive: K_ij grad log p(theta_j)
        acc += (2.0 / h) * (Theta - Theta[j]) * kj   # repulsive: grad_{theta_j} K_ij
    return acc / n


def svgd_step(Theta, G, step_size, rule=BW_MEDIAN_LN_N, h_fixed=1.0):
    """One Jacobi SVGD step.  Returns (Theta_new, info) with info = {D, h, K, phi}."""
    Theta = np.asarray(Theta, dtype=np.float64)
    D = sq_dists(Theta)
    h = bandwidth(D, rule, h_fixed)
    K = kernel_matrix(D, h)
    ph = phi(Theta, G, K, h)
    return Theta + step_size * ph, {"D": D, "h": h, "K": K, "phi": ph}


def svgd_run(Theta0, dims, batches, steps, step_size, act="tanh", lik_scale=1.0,
             prior="uniform", sigma=1.0, rule=BW_MEDIAN_LN_N, h_fixed=1.0):
    """Algorithm of PAPER.md:643-664 (Fig. supp:svgd) with our readings:
    per step: g_i for every particle (pstep), then the SVGD update (psend SVGD_UPDATE).

    `batches(t)` returns the (x, y) batch for step t.  Records the pre-update
    mean loss over particles and particle 0's loss (R19).
    Returns (Theta_T, mean_losses, loss0s, hs)."""
    Theta = np.asarray(Theta0, dtype=np.float64).copy()
    mean_l, l0, hs = [], [], []
    for t in range(steps):
        x, y = batches(t)
        G, losses = mlp.grads_all(Theta, dims, x, y, act=act, lik_scale=lik_scale,
                                  prior=prior, sigma=sigma)
        Theta, info = svgd_step(Theta, G, step_size, rule, h_fixed)
        mean_l.append(float(losses.mean()))
        l0.append(float(losses[0]))
        hs.append(info["h"])
    return Theta, np.array(mean_l), np.array(l0), np.array(hs)
