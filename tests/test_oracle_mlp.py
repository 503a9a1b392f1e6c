"""Pins for oracle.mlp: worked examples, closed forms and finite differences
(PAPER.md:152-157, 662)."""
import math
import os

import numpy as np
import pytest

from oracle import mlp

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold():
    out = {}
    with open(os.path.join(GOLD, "spec_examples.txt")) as f:
        for ln in f:
            if ln.strip() and not ln.startswith("#"):
                parts = [p.strip() for p in ln.split("|")]
                out[parts[0]] = float(parts[2])
    return out


def test_mse_worked_examples():
    g = _gold()
    assert mlp.mse(np.array([[0.0]]), np.array([[2.0]])) == g["mse"]
    y = np.random.default_rng(0).standard_normal((5, 2))
    assert mlp.mse(y, y) == g["mse_equal"]


def test_prior_worked_examples():
    g = _gold()
    th = np.full(7, 8.0)
    assert np.all(mlp.prior_grad(th, "gaussian", 2.0) == g["prior_gauss"])
    assert np.all(mlp.prior_grad(th, "uniform") == g["prior_uniform"])
    # linear in theta
    r = np.random.default_rng(1).standard_normal(11)
    assert np.allclose(mlp.prior_grad(3.0 * r, "gaussian", 1.5), 3.0 * mlp.prior_grad(r, "gaussian", 1.5))


def test_forward_special_cases():
    dims = (3, 5, 4, 2)
    d = sum(dims[l] * dims[l + 1] + dims[l + 1] for l in range(3))
    x = np.random.default_rng(2).standard_normal((6, 3))
    _, _, yhat = mlp.forward(np.zeros(d), dims, x)
    assert np.all(yhat == 0.0)
    # 1-layer identity net W = I, b = 0 -> yhat = x
    theta = np.concatenate([np.eye(2).ravel(), np.zeros(2)])
    _, _, yhat = mlp.forward(theta, (2, 2), np.array([[1.0, 2.0]]))
    assert np.array_equal(yhat, np.array([[1.0, 2.0]]))


def test_forward_hand_set_two_layer_tanh():
    # dims [1,1,1]: W1=0.5, b1=0.25, W2=2, b2=1, x=1 -> 2*tanh(0.75)+1 (scalar evaluation)
    theta = np.array([0.5, 0.25, 2.0, 1.0])
    _, _, yhat = mlp.forward(theta, (1, 1, 1), np.array([[1.0]]))
    assert yhat[0, 0] == pytest.approx(2.0 * math.tanh(0.75) + 1.0, rel=0, abs=1e-15)
    # 2-wide hidden layer, evaluated scalar by scalar
    W1 = [[0.3], [-0.7]]; b1 = [0.1, 0.2]; W2 = [[1.5, -0.5]]; b2 = [0.05]
    theta = np.array([W1[0][0], W1[1][0], b1[0], b1[1], W2[0][0], W2[0][1], b2[0]])
    x = 0.9
    h0 = math.tanh(W1[0][0] * x + b1[0]); h1 = math.tanh(W1[1][0] * x + b1[1])
    expect = W2[0][0] * h0 + W2[0][1] * h1 + b2[0]
    _, _, yhat = mlp.forward(theta, (1, 2, 1), np.array([[x]]))
    assert yhat[0, 0] == pytest.approx(expect, abs=1e-15)


def test_linear_net_closed_form_gradient():
    # single Linear layer + MSE: dW = (2/(B d_out)) (Wx+b-y)^T x, db = (2/(B d_out)) sum (Wx+b-y)
    rng = np.random.default_rng(3)
    d_in, d_out, B = 4, 3, 7
    W = rng.standard_normal((d_out, d_in)); b = rng.standard_normal(d_out)
    x = rng.standard_normal((B, d_in)); y = rng.standard_normal((B, d_out))
    theta = np.concatenate([W.ravel(), b])
    loss, g = mlp.mse_grad(theta, (d_in, d_out), x, y)
    r = x @ W.T + b - y
    assert loss == pytest.approx(float((r ** 2).sum() / (B * d_out)), rel=1e-14)
    dW = 2.0 / (B * d_out) * (r.T @ x)
    db = 2.0 / (B * d_out) * r.sum(0)
    assert np.allclose(g, np.concatenate([dW.ravel(), db]), rtol=1e-13, atol=1e-15)
    # single datapoint: 2 x^T (W x - y) / batch
    loss1, g1 = mlp.mse_grad(theta, (d_in, d_out), x[:1], y[:1])
    r1 = x[0] @ W.T + b - y[0]
    assert np.allclose(g1[:d_in * d_out].reshape(d_out, d_in), 2.0 * np.outer(r1, x[0]) / d_out)


def test_zero_residual_gives_zero_grads():
    # yhat == y exactly -> loss and every gradient are zero (loss constant at its minimum)
    rng = np.random.default_rng(4)
    dims = (2, 5, 1)
    theta = rng.standard_normal(2 * 5 + 5 + 5 + 1)
    x = rng.standard_normal((9, 2))
    _, _, yhat = mlp.forward(theta, dims, x)
    loss, g = mlp.mse_grad(theta, dims, x, yhat.copy())
    assert loss == 0.0 and np.all(g == 0.0)


def _fd_check(theta, dims, x, y, act, h=1e-5):
    loss, g = mlp.mse_grad(theta, dims, x, y, act)
    for k in range(theta.size):
        tp = theta.copy(); tp[k] += h
        tm = theta.copy(); tm[k] -= h
        fd = (mlp.mse(mlp.forward(tp, dims, x, act)[2], y) - mlp.mse(mlp.forward(tm, dims, x, act)[2], y)) / (2 * h)
        assert abs(fd - g[k]) <= 1e-5 * abs(fd) + 1e-8, (k, fd, g[k])


@pytest.mark.parametrize("seed", range(50))
def test_backprop_matches_central_differences(seed):
    """every component within 1e-5 rel (1e-8 abs floor), nets <= 4 layers, dims <= 8."""
    rng = np.random.default_rng(100 + seed)
    L = int(rng.integers(1, 5))
    dims = tuple(int(v) for v in rng.integers(1, 9, size=L + 1))
    act = ("tanh", "identity", "relu")[seed % 3]
    d = sum(dims[l] * dims[l + 1] + dims[l + 1] for l in range(L))
    theta = rng.standard_normal(d) * 0.7
    B = int(rng.integers(1, 6))
    x = rng.standard_normal((B, dims[0])); y = rng.standard_normal((B, dims[-1]))
    _fd_check(theta, dims, x, y, act)


def test_grad_log_post_sign_and_scale():
    # g = -lambda grad MSE + grad log p0 is an ascent direction on log p (R7/R9)
    rng = np.random.default_rng(7)
    dims = (2, 6, 6, 1)
    d = 2 * 6 + 6 + 36 + 6 + 6 + 1
    theta = rng.standard_normal(d) * 0.5
    x = rng.standard_normal((16, 2)); y = np.sin(x[:, :1])
    g1, loss = mlp.grad_log_post(theta, dims, x, y, lik_scale=1.0)
    g3, _ = mlp.grad_log_post(theta, dims, x, y, lik_scale=3.0)
    assert np.allclose(g3, 3.0 * g1)
    t = 1e-3
    assert mlp.mse(mlp.forward(theta + t * g1, dims, x)[2], y) < loss
    gg, _ = mlp.grad_log_post(theta, dims, x, y, lik_scale=2.0, prior="gaussian", sigma=0.5)
    assert np.allclose(gg, 2.0 * g1 - theta / 0.25)
