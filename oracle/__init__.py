"""ORACLE — test infrastructure, not product code.

A plain, slow, obviously-correct float64 CPU implementation of PusH's SVGD
particle step (arXiv 2306.06528), written from the paper:

* ``oracle.mlp``   — per-particle MLP forward, MSE loss, hand-written backprop,
                     prior gradient, g = grad log p (Eq. eq:grad).
* ``oracle.svgd``  — pairwise squared distances, median-heuristic bandwidth,
                     RBF kernel matrix, the SVGD direction
                     phi(theta_i) = (1/n) sum_j [K_ij grad log p(theta_j) + grad_{theta_j} K_ij]
                     and the Jacobi step (Fig. supp:svgd; north star).
* ``oracle.svgd_paper`` — PusH's own update of the listing (per-tensor kernel, 1/n on the
                     repulsion only, unweighted prior; NEXT-2).
* ``oracle.init``  — the counter-based K0 initialiser (SplitMix64; R14).
* ``oracle.swag``  — deep-ensemble step and diagonal SWAG moments / samples (NEXT-3).
* ``oracle.predict`` — predictive pushforward: per-particle outputs, cross-particle mean and
                     population std.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The CUDA path shares no code
with it (no kernels, headers, helpers or constant generators).

Pins: every function is checked by ``tests/test_oracle_*.py`` (-m "not gpu")
against closed forms, finite differences, special cases and brute force.
Functions without such a pin are marked "parity unpinned" (none at present;
see DESIGN.md §Oracle).
"""
from . import init, mlp, predict, svgd, svgd_paper, swag  # noqa: F401
