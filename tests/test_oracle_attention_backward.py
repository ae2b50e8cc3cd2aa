"""Pins of the attention-backward oracle (oracle/attention_backward.py, NEXT-1 partial) against what
the mathematics fixes: central finite differences of the forward (a separate code path), the closed
forms of a one-row history and of zero queries, and request-level aggregation: the gradient
a request's shared history receives from all its targets at once equals the sum of the gradients of
single-target requests over the same history."""
import numpy as np

from oracle import attention_backward as ab


def _case(rng, lengths, rows, d=8, scale=1.0):
    T, NQ = int(sum(lengths)), int(sum(rows))
    U = scale * rng.standard_normal((NQ, d))
    Xt = rng.standard_normal((T, d))
    dY = rng.standard_normal((NQ, d))
    q_off = np.concatenate([[0], np.cumsum(rows)]).astype(int)
    return U, Xt, dY, q_off


def test_finite_differences():
    rng = np.random.default_rng(0)
    lengths, rows = [5, 1, 9], [3, 2, 0]
    U, Xt, dY, q_off = _case(rng, lengths, rows, scale=0.7)
    dX, dU = ab.backward(U, Xt, dY, lengths, q_off)
    loss = lambda U_, X_: float((dY * ab.forward(U_, X_, lengths, q_off)).sum())
    h = 1e-6
    for arr, grad, name in ((Xt, dX, "dX"), (U, dU, "dU")):
        num = np.zeros_like(arr)
        for idx in np.ndindex(arr.shape):
            p, m = arr.copy(), arr.copy()
            p[idx] += h
            m[idx] -= h
            num[idx] = (loss(p, Xt) - loss(m, Xt)) / (2 * h) if name == "dU" else (loss(U, p) - loss(U, m)) / (2 * h)
        assert np.abs(num - grad).max() <= 1e-7 * max(1.0, np.abs(grad).max()), name


def test_single_history_row_closed_form():
    """L_b = 1: alpha = 1 for every query row, so dX~ = sum of the request's dY rows and dU = 0."""
    rng = np.random.default_rng(1)
    U, Xt, dY, q_off = _case(rng, [1], [4])
    dX, dU = ab.backward(U, Xt, dY, [1], q_off)
    assert np.allclose(dX[0], dY.sum(0), atol=1e-14)
    assert np.abs(dU).max() <= 1e-14


def test_zero_queries_mean_pooling():
    """U = 0: alpha = 1/L (mean pooling, P6), so dX~_j = (sum of dY rows) / L for every row j."""
    rng = np.random.default_rng(2)
    U, Xt, dY, q_off = _case(rng, [6], [3])
    U[:] = 0
    dX, dU = ab.backward(U, Xt, dY, [6], q_off)
    assert np.allclose(dX, np.tile(dY.sum(0) / 6, (6, 1)), atol=1e-14)


def test_request_level_aggregation():
    """One request with m query rows == m single-row requests over copies of the same history, their
    history gradients summed (and identical dU)."""
    rng = np.random.default_rng(3)
    L, m, d = 7, 5, 8
    U, Xt, dY, q_off = _case(rng, [L], [m], d=d)
    dX, dU = ab.backward(U, Xt, dY, [L], q_off)
    Xrep = np.tile(Xt, (m, 1))
    dXs, dUs = ab.backward(U, Xrep, dY, [L] * m, np.arange(m + 1))
    assert np.allclose(dX, dXs.reshape(m, L, d).sum(0), atol=1e-12)
    assert np.allclose(dU, dUs, atol=1e-12)
