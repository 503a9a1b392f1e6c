"""ORACLE (test infrastructure) — deep ensembles and diagonal SWAG on the particle substrate
(SURVEY.md §8(f) NEXT-3).

Passages followed
-----------------
* Deep ensemble (Fig. lang:de): every particle takes its own optimiser step on its own
  loss; with plain gradient steps on log p this is theta_i <- theta_i + eps * g_i (SVGD with K = I and no
  repulsion).
* SWAG (Fig. supp:swag): streaming moments
      mean <- (mean * n + theta) / (n + 1),   mom2 <- (mom2 * n + theta^2) / (n + 1),   n <- n + 1,
  started from one snapshot with n = 1 (R22: mom2 starts at theta_0^2), and the diagonal
  Gaussian sample theta_s = mean + sqrt(max(mom2 - mean^2, 0)) * z.
* z ~ N(0, 1) by Box-Muller on a counter-based stream (push.h, push_swag_sample):
  u1 = (m1 + 1) 2^-24, u2 = m2 2^-24, m = top 24 bits of mix64(seed ^ mix64(2 ((i << 32) | k) + {0, 1})),
  z = sqrt(-2 ln u1) cos(2 pi u2).  The random numbers are part of the method's inputs, generated here
  in float64 from the same counters the CUDA side uses.
Pins: tests/test_oracle_swag.py.
"""
from __future__ import annotations

import numpy as np

from .init import mix64


def ensemble_step(Theta, G, eps):
    """theta_i + eps * g_i for every particle."""
    return np.asarray(Theta, dtype=np.float64) + eps * np.asarray(G, dtype=np.float64)


def swag_moments(snapshots):
    """(mean, mom2, n) after streaming every snapshot in order."""
    first = np.asarray(snapshots[0], dtype=np.float64)
    mean, mom2, n = first.copy(), first * first, 1
    for th in snapshots[1:]:
        th = np.asarray(th, dtype=np.float64)
        mean = (mean * n + th) / (n + 1)
        mom2 = (mom2 * n + th * th) / (n + 1)
        n += 1
    return mean, mom2, n


def swag_normal(seed: int, row0: int, rows: int, d: int):
    """z[r][k] for global particle rows row0..row0+rows-1 and canonical indices k < d."""
    k = np.arange(d, dtype=np.uint64)
    z = np.empty((rows, d))
    s = np.uint64(seed)
    for r in range(rows):
        with np.errstate(over="ignore"):
            ctr = ((np.uint64(row0 + r) << np.uint64(32)) | k) * np.uint64(2)
            m1 = mix64(s ^ mix64(ctr)) >> np.uint64(40)
            m2 = mix64(s ^ mix64(ctr + np.uint64(1))) >> np.uint64(40)
        u1 = (m1.astype(np.float64) + 1.0) * 2.0 ** -24
        u2 = m2.astype(np.float64) * 2.0 ** -24
        z[r] = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return z


def swag_sample(mean, mom2, z):
    """Diagonal SWAG draw."""
    mean = np.asarray(mean, dtype=np.float64)
    return mean + np.sqrt(np.maximum(np.asarray(mom2, dtype=np.float64) - mean * mean, 0.0)) * z
