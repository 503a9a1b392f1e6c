"""ORACLE (test infrastructure) — counter-based particle initialisation (K0).

The paper says nothing about initialisation beyond `pinit` creating an
instance of g(.; theta_i) (§2.2).  SPEC.md:126 reads it as
"per-layer uniform in +-1/sqrt(d_in), seeded"; the RNG is fixed by
DESIGN.md reading R14:

    m          = mix64(seed XOR mix64((i << 32) | k)) >> 40     (24 bits)
    u          = m * 2^-24
    theta_ik   = fp32(2u - 1) * fp32(1 / sqrt(fan_in))          (one fp32 multiply)

where mix64 is the SplitMix64 output function *including* the +gamma add,
k is the canonical flat index of the parameter inside the particle, and
fan_in is in_l of k's layer (a bias uses its own layer's in_l).

Pinned by tests/test_oracle_init.py: SplitMix64 known answers
(tests/golden/splitmix64.txt) and the three init known answers of
SURVEY.md App. A.
"""
from __future__ import annotations

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z):
    """SplitMix64 output function incl. the +gamma increment (vectorised, wraps mod 2^64)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def layer_fan_in(dims):
    """fan_in of every canonical flat index (weight then bias per layer, torch (out,in))."""
    parts = []
    for l in range(len(dims) - 1):
        n_in, n_out = dims[l], dims[l + 1]
        parts.append(np.full(n_in * n_out + n_out, n_in, dtype=np.int64))
    return np.concatenate(parts)


def init_theta(n: int, dims, seed: int) -> np.ndarray:
    """Initial particle matrix Theta [n, d] (float32) per DESIGN.md R14."""
    fan = layer_fan_in(dims)
    d = fan.size
    k = np.arange(d, dtype=np.uint64)
    out = np.empty((n, d), dtype=np.float32)
    seed64 = np.uint64(seed)
    for i in range(n):
        ctr = (np.uint64(i) << np.uint64(32)) | k
        m = mix64(seed64 ^ mix64(ctr)) >> np.uint64(40)
        u = m.astype(np.float64) * 2.0 ** -24
        two_u_m1 = (2.0 * u - 1.0).astype(np.float32)      # exact: 24-bit numerator
        bound = (1.0 / np.sqrt(fan.astype(np.float64))).astype(np.float32)
        out[i] = two_u_m1 * bound                          # single fp32 rounding
    return out
