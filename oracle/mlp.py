"""ORACLE (test infrastructure) — per-particle MLP, MSE loss, hand-written backprop,
prior gradient and the posterior-gradient g = grad log p(theta | D), in float64.

Passages followed
-----------------
* Posterior-gradient principle, PAPER.md:152-157 (§2.2, Eq. eq:grad):
      grad log p(theta_i | D) = grad log( p(D | theta_i) p(theta_i) )
  With the likelihood read as exp(-lambda * MSE) (R9)
  and p0 the prior:  g_i = -lambda * grad MSE_i + grad log p0(theta_i).
* Loss: torch.nn.MSELoss() mean reduction, PAPER.md:662 (Fig. supp:svgd);
  SPEC.md:72 "mean over all elements of squared difference".
* The network: a stack of fully connected layers, PAPER.md:355 (§4.2) — our
  dims list [d_in, H, ..., d_out]; hidden activation tanh by default (R13),
  output layer identity.
* Canonical flat layout (R15): for l = 1..L, W_l as [out_l][in_l] row-major
  (torch nn.Linear), then b_l[out_l] — module.parameters() order.
* Priors: Uniform -> 0; Gaussian(sigma) -> -theta / sigma^2.

Everything here is plain numpy float64; matmul (a library primitive) is the
only building block.  Pins: tests/test_oracle_mlp.py.
"""
from __future__ import annotations

import numpy as np

ACTS = ("tanh", "relu", "identity")


def unpack(theta, dims):
    """Split a flat canonical parameter vector into [(W_l [out,in], b_l [out])]."""
    theta = np.asarray(theta, dtype=np.float64)
    layers, off = [], 0
    for l in range(len(dims) - 1):
        n_in, n_out = dims[l], dims[l + 1]
        W = theta[off:off + n_in * n_out].reshape(n_out, n_in)
        off += n_in * n_out
        b = theta[off:off + n_out]
        off += n_out
        layers.append((W, b))
    assert off == theta.size, (off, theta.size)
    return layers


def pack(layers):
    return np.concatenate([np.concatenate([W.ravel(), b.ravel()]) for W, b in layers])


def _act(z, act):
    if act == "tanh":
        return np.tanh(z)
    if act == "relu":
        return np.maximum(z, 0.0)
    if act == "identity":
        return z
    raise ValueError(act)


def _act_deriv(z, a, act):
    """sigma'(z) expressed as tanh' = 1 - a^2, relu'(z) = [z > 0] (relu'(0) = 0, R13)."""
    if act == "tanh":
        return 1.0 - a * a
    if act == "relu":
        return (z > 0.0).astype(np.float64)
    if act == "identity":
        return np.ones_like(z)
    raise ValueError(act)


def forward(theta, dims, x, act="tanh"):
    """a_0 = x; z_l = a_{l-1} W_l^T + b_l; a_l = sigma(z_l) (l < L); yhat = z_L.

    Returns (zs, activations, yhat) where activations[0] = x."""
    layers = unpack(theta, dims)
    a = np.asarray(x, dtype=np.float64)
    acts, zs = [a], []
    L = len(layers)
    for l, (W, b) in enumerate(layers):
        z = a @ W.T + b
        zs.append(z)
        a = _act(z, act) if l < L - 1 else z
        acts.append(a)
    return zs, acts, acts[-1]


def mse(yhat, y):
    """torch.nn.MSELoss() (mean over all B*d_out elements)."""
    yhat = np.asarray(yhat, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    return float(np.mean((yhat - y) ** 2))


def mse_grad(theta, dims, x, y, act="tanh"):
    """(loss, grad of the mean MSE w.r.t. the flat theta) by reverse-mode backprop.

    delta_L = 2 (yhat - y) / (B d_out); for l = L..1:
        dW_l = delta_l^T a_{l-1};  db_l = sum_b delta_l;
        delta_{l-1} = (delta_l W_l) * sigma'(z_{l-1})   (l > 1)."""
    layers = unpack(theta, dims)
    zs, acts, yhat = forward(theta, dims, x, act)
    y = np.asarray(y, dtype=np.float64)
    B, d_out = yhat.shape
    loss = float(np.mean((yhat - y) ** 2))
    delta = 2.0 * (yhat - y) / (B * d_out)
    grads = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        W, _ = layers[l]
        dW = delta.T @ acts[l]
        db = delta.sum(axis=0)
        grads[l] = (dW, db)
        if l > 0:
            delta = (delta @ W) * _act_deriv(zs[l - 1], acts[l], act)
    return loss, pack(grads)


def prior_grad(theta, prior="uniform", sigma=1.0):
    """grad log p0(theta): Uniform -> 0, Gaussian(sigma) -> -theta / sigma^2."""
    theta = np.asarray(theta, dtype=np.float64)
    if prior == "uniform":
        return np.zeros_like(theta)
    if prior == "gaussian":
        return -theta / (sigma * sigma)
    raise ValueError(prior)


def grad_log_post(theta, dims, x, y, act="tanh", lik_scale=1.0, prior="uniform", sigma=1.0):
    """g = grad log p(theta | D) = -lambda grad MSE + grad log p0   (Eq. eq:grad).

    Returns (g, loss)."""
    loss, gmse = mse_grad(theta, dims, x, y, act)
    return -lik_scale * gmse + prior_grad(theta, prior, sigma), loss


def grads_all(Theta, dims, x, y, **kw):
    """Per-particle g_i for every row of Theta (particles are independent)."""
    Theta = np.asarray(Theta, dtype=np.float64)
    G = np.empty_like(Theta)
    losses = np.empty(Theta.shape[0])
    for i in range(Theta.shape[0]):
        G[i], losses[i] = grad_log_post(Theta[i], dims, x, y, **kw)
    return G, losses
