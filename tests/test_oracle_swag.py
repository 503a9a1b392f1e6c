"""Pins of oracle.swag (deep ensembles and diagonal SWAG)."""
import numpy as np

from oracle import svgd as osvgd
from oracle import swag as oswag


def test_ensemble_step_equals_single_particle_svgd():
    rng = np.random.default_rng(0)
    th, g = rng.standard_normal((1, 7)), rng.standard_normal((1, 7))
    ref, _ = osvgd.svgd_step(th, g, 0.05)       # n = 1: SVGD is gradient ascent
    np.testing.assert_allclose(oswag.ensemble_step(th, g, 0.05), ref, rtol=0, atol=1e-15)


def test_streaming_moments_equal_snapshot_statistics():
    rng = np.random.default_rng(1)
    snaps = [rng.standard_normal((3, 11)) for _ in range(9)]
    mean, mom2, n = oswag.swag_moments(snaps)
    assert n == 9
    np.testing.assert_allclose(mean, np.mean(snaps, axis=0), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(mom2, np.mean(np.square(snaps), axis=0), rtol=1e-12, atol=1e-14)


def test_constant_parameters_have_zero_variance_and_sample_the_mean():
    th = np.random.default_rng(2).standard_normal((2, 5))
    mean, mom2, _ = oswag.swag_moments([th, th, th])
    z = oswag.swag_normal(7, 0, 2, 5)
    np.testing.assert_allclose(oswag.swag_sample(mean, mom2, z), th, rtol=0, atol=1e-15)


def test_counter_normals_are_standard_normal_and_deterministic():
    z = oswag.swag_normal(123, 0, 4, 100_000).ravel()
    assert abs(z.mean()) < 5 / np.sqrt(z.size)
    assert abs(z.var() - 1.0) < 5 * np.sqrt(2.0 / z.size)
    assert abs(np.mean(np.abs(z) < 1.0) - 0.682689) < 0.005
    np.testing.assert_array_equal(oswag.swag_normal(123, 2, 1, 50), oswag.swag_normal(123, 0, 4, 50)[2:3])
    assert not np.array_equal(oswag.swag_normal(124, 0, 1, 50), oswag.swag_normal(123, 0, 1, 50))
