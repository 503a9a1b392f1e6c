"""Pins for oracle.init (R14): SplitMix64 known answers and the K0 KATs."""
import os

import numpy as np

from oracle import init as oinit

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def test_splitmix64_known_answers():
    gamma = 0x9E3779B97F4A7C15
    for k, hexv in _rows("splitmix64.txt"):
        state = ((int(k) - 1) * gamma) % 2 ** 64
        assert int(oinit.mix64(np.uint64(state))) == int(hexv, 16)


def test_init_known_answers():
    for seed, i, k, m, v in _rows("init_kat.txt"):
        seed, i, k = int(seed), int(i), int(k)
        ctr = np.uint64((i << 32) | k)
        mm = int(oinit.mix64(np.uint64(seed) ^ oinit.mix64(ctr)) >> np.uint64(40))
        if m != "-":
            assert mm == int(m)
        two_u_m1 = np.float32(2.0 * (mm * 2.0 ** -24) - 1.0)
        assert two_u_m1 == np.float32(v)


def test_init_theta_matches_kat_and_bounds():
    dims = (1, 32, 32, 1)
    th = oinit.init_theta(4, dims, seed=0)
    assert th.dtype == np.float32 and th.shape == (4, 1153)
    # theta_00: layer 1 (fan_in = 1) -> bound 1
    assert th[0, 0] == np.float32(0.30489695) * np.float32(1.0)
    assert th[0, 1] == np.float32(-0.26362097)
    assert th[1, 0] == np.float32(0.4996649)
    # per-layer bound 1/sqrt(fan_in)
    fan = oinit.layer_fan_in(dims)
    bound = (1.0 / np.sqrt(fan)).astype(np.float32)
    assert np.all(np.abs(th) <= bound[None, :])
    # layer 2 entries are spread over the whole +-1/sqrt(32) range, mean ~ 0
    seg = th[:, 64:64 + 32 * 32]
    assert abs(seg.mean()) < 0.02 and seg.max() > 0.9 / np.sqrt(32) and seg.min() < -0.9 / np.sqrt(32)


def test_init_deterministic_and_seeded():
    a = oinit.init_theta(3, (2, 8, 1), seed=5)
    b = oinit.init_theta(3, (2, 8, 1), seed=5)
    c = oinit.init_theta(3, (2, 8, 1), seed=6)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)
    # rows are distinct particles
    assert not np.array_equal(a[0], a[1])
