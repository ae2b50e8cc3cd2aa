"""Pins of the history-path backward oracle (oracle/history_backward.py, NEXT-1 partial): central finite
differences of the C oracle's own forward, LN(SwiGLUFFN(X)) (oracle.swigluffn / oracle.layernorm, pinned in
test_oracle_pins.py), for every input and weight, plus two closed forms (LN's gradient is orthogonal to the
constant and to x^ directions: sum_e dy_e = 0 and dbeta = column sums of dX~)."""
import numpy as np

import oracle
from oracle import history_backward as hb


def _loss(X, Wu, Wv, Wo, g, b, dXt):
    return float((dXt * oracle.layernorm(oracle.swigluffn(X, Wu, Wv, Wo), g, b)).sum())


def test_finite_differences():
    rng = np.random.default_rng(0)
    n, d, rd = 3, 4, 6
    X = rng.standard_normal((n, d))
    Wu, Wv = rng.standard_normal((d, rd)) / 2, rng.standard_normal((d, rd)) / 2
    Wo = rng.standard_normal((rd, d)) / 2
    g, b = 1 + 0.1 * rng.standard_normal(d), 0.1 * rng.standard_normal(d)
    dXt = rng.standard_normal((n, d))
    grads = dict(zip(["X", "Wu", "Wv", "Wo", "g", "b"], hb.backward(X, Wu, Wv, Wo, g, b, dXt)))
    args = dict(X=X, Wu=Wu, Wv=Wv, Wo=Wo, g=g, b=b)
    h = 1e-6
    for name, arr in args.items():
        num = np.zeros_like(arr)
        for idx in np.ndindex(arr.shape):
            p, m = dict(args), dict(args)
            p[name] = arr.copy()
            m[name] = arr.copy()
            p[name][idx] += h
            m[name][idx] -= h
            num[idx] = (_loss(dXt=dXt, **p) - _loss(dXt=dXt, **m)) / (2 * h)
        got = grads[name].reshape(arr.shape)
        assert np.abs(num - got).max() <= 1e-6 * max(1.0, np.abs(got).max()), name


def test_layernorm_gradient_invariants():
    rng = np.random.default_rng(1)
    n, d, rd = 5, 8, 16
    X = rng.standard_normal((n, d))
    Wu, Wv, Wo = rng.standard_normal((d, rd)), rng.standard_normal((d, rd)), rng.standard_normal((rd, d))
    dXt = rng.standard_normal((n, d))
    dX, dWu, dWv, dWo, dg, db = hb.backward(X, Wu, Wv, Wo, np.ones(d), np.zeros(d), dXt)
    assert np.allclose(db, dXt.sum(0), atol=1e-12)
    # the gradient reaching y has zero row sums (LN removes the mean direction), so dWo = H^T dy has zero
    # row sums as well
    assert np.allclose(dWo.sum(1), 0.0, atol=1e-9)
