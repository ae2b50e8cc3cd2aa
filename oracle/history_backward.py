"""Oracle of the history-path backward (partial) -- TEST INFRASTRUCTURE ONLY.

Only tests/ may import this module; the product path (paper_2511_06077_b200/) never does.  Plain
numpy, float64, the textbook backward of one layer's history encoding, Eq.(1)-(2):

    a = X Wu,  g = X Wv,  H = a * silu(g),  y = H Wo,  X~ = (y - mu) / sqrt(var + eps) * gamma + beta

(readings R1-R3: SiLU gate on Wv, no biases, biased variance, eps inside the root).  Given dX~:

    x^ = (y - mu) / s,                  dgamma = sum_rows dX~ * x^,   dbeta = sum_rows dX~
    dx^ = dX~ * gamma,                  dy = (dx^ - mean(dx^) - x^ * mean(dx^ * x^)) / s
    dWo = H^T dy,                       dH = dy Wo^T
    da = dH * silu(g),                  dg = dH * a * silu'(g),  silu'(g) = sig(g) (1 + g (1 - sig(g)))
    dWu = X^T da,  dWv = X^T dg,        dX = da Wu^T + dg Wv^T

The rows are the kept history rows of a projection; under RLB each row appears once per request,
however many targets share it, so these gradients are already aggregated at the request level
(P:L396).  Pinned in tests/test_oracle_history_backward.py by central finite differences of
oracle.swigluffn / oracle.layernorm (the forward the oracle already pins).
"""
from __future__ import annotations

import numpy as np


def backward(X, Wu, Wv, Wo, gamma, beta, dXt, eps: float = 1e-5):
    """(dX, dWu, dWv, dWo, dgamma, dbeta) for one layer; all float64."""
    X, Wu, Wv, Wo, dXt = (np.asarray(a, np.float64) for a in (X, Wu, Wv, Wo, dXt))
    gamma = np.asarray(gamma, np.float64).reshape(-1)
    a = X @ Wu
    g = X @ Wv
    sig = 1.0 / (1.0 + np.exp(-g))
    H = a * g * sig
    y = H @ Wo
    mu = y.mean(1, keepdims=True)
    s = np.sqrt(((y - mu) ** 2).mean(1, keepdims=True) + eps)
    xh = (y - mu) / s
    dgamma = (dXt * xh).sum(0)
    dbeta = dXt.sum(0)
    dxh = dXt * gamma
    dy = (dxh - dxh.mean(1, keepdims=True) - xh * (dxh * xh).mean(1, keepdims=True)) / s
    dWo = H.T @ dy
    dH = dy @ Wo.T
    da = dH * g * sig
    dg = dH * a * sig * (1.0 + g * (1.0 - sig))
    dWu = X.T @ da
    dWv = X.T @ dg
    dX = da @ Wu.T + dg @ Wv.T
    return dX, dWu, dWv, dWo, dgamma, dbeta
