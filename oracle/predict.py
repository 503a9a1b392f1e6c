"""ORACLE (test infrastructure) — predictive pushforward of the particle approximation.

Passages followed
-----------------
* PAPER.md:128-146 (§2.2): the particles theta_1..theta_n approximate the pushforward of mu through
  g(x; .); `ppush(mu)(g(x; .))` is the set of per-particle functions {g(x; theta_i)}.
* SPEC.md:368-376 (`ppush_predict`): per-particle outputs on a grid, plus their cross-particle mean and
  population standard deviation (the uncertainty of the posterior predictive).

Plain float64 numpy on top of oracle.mlp.forward.  Pins: tests/test_oracle_predict.py.
"""
from __future__ import annotations

import numpy as np

from . import mlp


def pushforward(Theta, dims, x, act="tanh"):
    """preds[i] = g(x; theta_i) for every particle (array [n, B, d_out])."""
    Theta = np.asarray(Theta, dtype=np.float64)
    return np.stack([mlp.forward(Theta[i], dims, x, act)[2] for i in range(Theta.shape[0])])


def predictive_summary(Theta, dims, x, act="tanh"):
    """(preds, mean, std): cross-particle mean and population std (ddof = 0) per input and output."""
    preds = pushforward(Theta, dims, x, act)
    return preds, preds.mean(axis=0), preds.std(axis=0)
