"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no MLP, no kernel, no SVGD
update): only data/target generators and random draws, all returned as
float32 numpy arrays.  The recipes are DESIGN.md "Input recipe" and
SURVEY.md §8(d) "Synthetic inputs":

* sine       (C1): x = -1 + 2b/(B-1), y = sin(2*pi*x)
* advection  (C2): (x,t) ~ U[0,1) x U[0,2], beta = 0.4,
                   u = 0.7 sin(2pi(x - beta t)) + 0.3 sin(6pi(x - beta t) + 1)
                   (PDEBench-Advection-shaped)
* burgers   (C3,S1): (x,t,nu) ~ U[-1,1] x U[0,1] x U[0.01,0.1],
                   Cole-Hopf closed form
                   u = 2 pi nu e^{-pi^2 nu t} sin(pi x) / (2 + e^{-pi^2 nu t} cos(pi x))
* random   (C4,C5): x ~ N(0, I), y = sin(x_1) + 0.1 N(0,1); 10 fixed batches
                   cycled ("random dataset with 10 batches")

Batch s always comes from np.random.default_rng(1000 + s).
"""
from __future__ import annotations

import numpy as np

N_RANDOM_BATCHES = 10


def batch(kind: str, B: int, d_in: int, d_out: int, step: int = 0):
    """Return (x [B, d_in], y [B, d_out]) float32 for generator `kind` at step `step`."""
    if kind == "sine":
        assert d_in == 1 and d_out == 1
        b = np.arange(B, dtype=np.float64)
        x = -1.0 + 2.0 * b / max(B - 1, 1)
        y = np.sin(2.0 * np.pi * x)
        return x.reshape(B, 1).astype(np.float32), y.reshape(B, 1).astype(np.float32)
    if kind == "random":
        rng = np.random.default_rng(1000 + (step % N_RANDOM_BATCHES))
        x = rng.standard_normal((B, d_in))
        y = np.sin(x[:, :1]) + 0.1 * rng.standard_normal((B, 1))
        y = np.repeat(y, d_out, axis=1)
        return x.astype(np.float32), y.astype(np.float32)
    rng = np.random.default_rng(1000 + step)
    if kind == "advection":
        assert d_in == 2 and d_out == 1
        xs = rng.uniform(0.0, 1.0, B)
        t = rng.uniform(0.0, 2.0, B)
        beta = 0.4
        s = xs - beta * t
        u = 0.7 * np.sin(2 * np.pi * s) + 0.3 * np.sin(6 * np.pi * s + 1.0)
        x = np.stack([xs, t], axis=1)
        return x.astype(np.float32), u.reshape(B, 1).astype(np.float32)
    if kind == "burgers":
        assert d_in == 3 and d_out == 1
        xs = rng.uniform(-1.0, 1.0, B)
        t = rng.uniform(0.0, 1.0, B)
        nu = rng.uniform(0.01, 0.1, B)
        e = np.exp(-np.pi ** 2 * nu * t)
        u = 2 * np.pi * nu * e * np.sin(np.pi * xs) / (2.0 + e * np.cos(np.pi * xs))
        x = np.stack([xs, t, nu], axis=1)
        return x.astype(np.float32), u.reshape(B, 1).astype(np.float32)
    if kind == "gauss":
        # generic regression: x ~ N(0,I), y = sum of sines (used for odd shapes in tests)
        x = rng.standard_normal((B, d_in))
        y = np.sin(x.sum(axis=1, keepdims=True)) * np.ones((1, d_out))
        return x.astype(np.float32), y.astype(np.float32)
    raise ValueError(f"unknown generator {kind!r}")


def workload_batch(w, step: int = 0):
    return batch(w.data, w.batch, w.dims[0], w.dims[-1], step)


def random_theta(n: int, d: int, seed: int, scale: float = 0.1):
    """Generic random particle matrix (float32), for kernel/update tests."""
    rng = np.random.default_rng(seed)
    return (scale * rng.standard_normal((n, d))).astype(np.float32)


def random_grads(n: int, d: int, seed: int, scale: float = 1.0):
    rng = np.random.default_rng(seed + 7919)
    return (scale * rng.standard_normal((n, d))).astype(np.float32)


def dyadic_theta(n: int, d: int, seed: int):
    """Entries k/8 with |k| <= 32 (SURVEY.md §8(c) 'Dyadic-lattice'): every squared
    distance is a multiple of 1/64 below 2^16 for d <= 2^10, hence exact in fp32."""
    assert d <= 1024
    rng = np.random.default_rng(seed)
    k = rng.integers(-32, 33, size=(n, d))
    return (k / 8.0).astype(np.float32)


def clustered_theta(n: int, d: int, seed: int, spread: float = 1e-2, center_scale: float = 1.0):
    """Particles clustered around a common centre: theta_i = mu + spread * delta_i (float32), the
    regime of a pretrained theta0 plus small noise or of particles that contracted during training
    (the Gram form of a7 must not cancel here)."""
    rng = np.random.default_rng(seed)
    mu = center_scale * rng.standard_normal(d)
    return (mu + spread * rng.standard_normal((n, d))).astype(np.float32)
