"""Pins of oracle.predict (predictive pushforward)."""
import numpy as np

from oracle import init as oinit
from oracle import mlp as omlp
from oracle import predict as opred


def test_single_particle_has_zero_spread_and_its_own_output():
    dims = [2, 8, 1]
    th = oinit.init_theta(1, dims, 3).astype(np.float64)
    x = np.random.default_rng(0).standard_normal((5, 2))
    preds, mean, std = opred.predictive_summary(th, dims, x)
    np.testing.assert_array_equal(mean, omlp.forward(th[0], dims, x)[2])
    assert np.all(std == 0.0)


def test_identical_particles_have_zero_spread():
    dims = [1, 4, 4, 2]
    th = np.tile(oinit.init_theta(1, dims, 1).astype(np.float64), (6, 1))
    x = np.linspace(-1, 1, 7).reshape(7, 1)
    _, mean, std = opred.predictive_summary(th, dims, x)
    # the mean of n equal values can differ from them by rounding: spread ~ one ulp of the mean
    assert np.all(std <= 4 * np.finfo(np.float64).eps * np.abs(mean).max())


def test_two_linear_particles_closed_form():
    # one identity Linear layer y = w x + b per particle: mean = (y1 + y2)/2, population std = |y1 - y2|/2
    dims = [1, 1]
    th = np.array([[2.0, 0.5], [-1.0, 1.5]])  # (w, b) per particle
    x = np.array([[-2.0], [0.0], [3.0]])
    preds, mean, std = opred.predictive_summary(th, dims, x, act="identity")
    y1, y2 = 2.0 * x + 0.5, -1.0 * x + 1.5
    np.testing.assert_allclose(preds[0], y1)
    np.testing.assert_allclose(mean, (y1 + y2) / 2)
    np.testing.assert_allclose(std, np.abs(y1 - y2) / 2)
