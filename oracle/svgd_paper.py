"""ORACLE (test infrastructure) — PusH's own SVGD update, float64.

Only tests/, __graft_entry__.smoke() and bench.py's baseline legs may import this module.

Passage followed: the listing `_svgd_update` of PAPER.md:609-641 (Fig. supp:svgd), line by line:

    acc = 0
    for j in range(n):
        grads = ppush(particles[j])                                   # PAPER.md:628-629  (prior of j)
        for idx, tmp in enumerate(acc):                               # PAPER.md:630      (per parameter TENSOR)
            k_ij = kernel(p_j[idx].flatten(), p_i[idx].flatten(), l)
            tmp += k_ij * p_j.grad[idx]                               # PAPER.md:633-634  (no 1/n)
            tmp += grads[idx]                                         # PAPER.md:635-636  (prior, unweighted)
            tmp += (1/n) * grad_arg1 kernel(p_j[idx], p_i[idx])       # PAPER.md:637-638  (1/n on repulsion)
    p_i -= lr * acc

Three switches (the `variant` bits of push_config, include/push.h) select these departures from the
canonical step (oracle.svgd) one at a time:

* per_tensor (PUSH_VAR_PER_TENSOR): the kernel is evaluated per parameter tensor
  (W_l and b_l of every layer, module.parameters() order; R15), with
  its own distances and, under a median rule, its own bandwidth.  Off: one tensor = all of theta.
* paper_norm (PUSH_VAR_PAPER_NORM, A5): drive terms weighted 1, repulsion 1/n.  Off: 1/n on both.
* prior_sum (PUSH_VAR_PRIOR_SUM, A8): G holds the likelihood term only and the prior gradients of
  all n particles are added unweighted, sum_j grad log p0(theta_j), with the drive weight.  Off: the
  prior is inside g_j and weighted by K_ij.

Readings kept from the canonical path: ascent on log p with g = -lambda grad MSE (A7, A9: the
listing's `p_j.grad` is the loss gradient and `p -= lr * acc` descends; we write both as ascent),
the repulsive sign grad_{theta_j} k(theta_j, theta_i) = (2/h)(theta_i - theta_j) k (A7),
K = exp(-r^2/h) so the paper's length scale l = 1 is h = 2 (A1), Jacobi simultaneity (A10),
j = i included (A11).  Pins: tests/test_oracle_svgd_paper.py.
"""
from __future__ import annotations

import numpy as np

from . import mlp, svgd


def tensor_ranges(dims):
    """[(offset, size)] of every parameter tensor in the canonical layout: W_l (out x in) then b_l
    (out) for l = 1..L (PAPER.md:560, 631 module.parameters() order; R15)."""
    out, off = [], 0
    for l in range(len(dims) - 1):
        w = dims[l] * dims[l + 1]
        out.append((off, w))
        off += w
        out.append((off, dims[l + 1]))
        off += dims[l + 1]
    return out


def svgd_step_variant(Theta, G, step_size, dims, per_tensor=True, paper_norm=True, prior_sum=True,
                      prior="uniform", sigma=1.0, rule=svgd.BW_FIXED, h_fixed=2.0):
    """One step of the listing for every particle i (Jacobi).  G: n x d, the likelihood term
    -lambda grad MSE if prior_sum else the whole grad log p.  Returns (Theta_new, info) with
    info = {"ranges", "D": [T x n x n], "h": [T], "K": [T x n x n]}."""
    Theta = np.asarray(Theta, dtype=np.float64)
    G = np.asarray(G, dtype=np.float64)
    n, d = Theta.shape
    ranges = tensor_ranges(dims) if per_tensor else [(0, d)]
    assert sum(s for _, s in ranges) == d
    w_drive = 1.0 if paper_norm else 1.0 / n
    w_rep = 1.0 / n
    # per tensor: distances, bandwidth and kernel
    Ds, hs, Ks = [], [], []
    for off, size in ranges:
        D = svgd.sq_dists(Theta[:, off:off + size])
        h = svgd.bandwidth(D, rule, h_fixed)
        Ds.append(D)
        hs.append(h)
        Ks.append(svgd.kernel_matrix(D, h))
    new = Theta.copy()
    for i in range(n):
        acc = np.zeros(d)
        for j in range(n):
            if prior_sum:
                pg = mlp.prior_grad(Theta[j], prior, sigma)          # grads = ppush(particles[j])
            for t, (off, size) in enumerate(ranges):
                sl = slice(off, off + size)
                k_ij = Ks[t][i, j]
                acc[sl] += w_drive * k_ij * G[j, sl]                  # tmp.add_(p_j.grad, alpha=k_ij)
                if prior_sum:
                    acc[sl] += w_drive * pg[sl]                       # tmp.add_(grads[idx])
                acc[sl] += w_rep * (2.0 / hs[t]) * (Theta[i, sl] - Theta[j, sl]) * k_ij  # grad_arg1, 1/n
        new[i] = Theta[i] + step_size * acc                           # p.add_(acc, alpha=-lr) as ascent
    return new, {"ranges": ranges, "D": np.array(Ds), "h": np.array(hs), "K": np.array(Ks)}
