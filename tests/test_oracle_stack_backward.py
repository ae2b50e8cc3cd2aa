"""Pins of the whole-stack backward oracle (oracle/stack_backward.py, NEXT-1) against what the mathematics
fixes, none of them by retyping its formulas:

* central finite differences of the C oracle's forward (oracle.forward, standard form Eq.(12), pinned in
  test_oracle_pins.py) over EVERY weight entry of every role and every input entry of a tiny stack
  (M = 3 layers, distinct weights per role, affine LayerNorms, a request without targets, an L_infer
  suffix that drops history rows) -- a dropped term, a wrong sign, index or transposed operand anywhere
  in the backward moves some entry;
* the module's own forward pass reproduces oracle.forward (Z and z);
* request-level aggregation: one request with m targets over a shared history has the gradients
  of m single-target requests over copies of that history, summed.
"""
import numpy as np

import oracle
import workload
from oracle import stack_backward as sb

D, H, R, M = 4, 2, 1, 3


def _weights(rng, d=D, r=R, M=M):
    w = {}
    for name, shape in workload.weight_shapes(d, r, M, shared_ffn=False, with_z=True).items():
        leaf = name.split(".")[-1]
        if leaf == "ln_g":
            w[name] = 1.0 + 0.2 * rng.standard_normal(shape)
        elif leaf == "ln_b":
            w[name] = 0.2 * rng.standard_normal(shape)
        else:
            w[name] = rng.standard_normal(shape) * (1.2 / np.sqrt(shape[0]))
    return w


def _case(seed=0):
    rng = np.random.default_rng(seed)
    w = _weights(rng)
    hist_off = np.array([0, 3, 4, 9])            # lengths 3, 1, 5
    tgt_off = np.array([0, 2, 2, 4])             # the middle request has no targets
    X = rng.standard_normal((9, D))
    xt = rng.standard_normal((4, D))
    dZ = rng.standard_normal((4, M, D))
    dz = rng.standard_normal((4, D))
    return w, X, hist_off, xt, tgt_off, dZ, dz


def _loss(w, X, hist_off, xt, tgt_off, dZ, dz, L_infer):
    Z, z = oracle.forward(w, d=D, h=H, r=R, M=M, X=X, hist_off=hist_off, xt=xt, tgt_off=tgt_off,
                          L_infer=L_infer, with_z=True, form=0)
    return float((dZ * Z).sum() + (dz * z).sum())


def test_finite_differences_every_entry():
    w, X, hist_off, xt, tgt_off, dZ, dz = _case()
    L_infer = 4  # request 2 keeps its last 4 of 5 rows: row 4 gets no gradient
    G, dX, dxt, _, _ = sb.backward(w, d=D, h=H, r=R, M=M, X=X, hist_off=hist_off, xt=xt, tgt_off=tgt_off,
                                   dZ=dZ, dz=dz, L_infer=L_infer)
    eps = 1e-6

    def fd(get, arr):
        num = np.zeros_like(arr)
        for idx in np.ndindex(arr.shape):
            keep = arr[idx]
            arr[idx] = keep + eps
            lp = get()
            arr[idx] = keep - eps
            lm = get()
            arr[idx] = keep
            num[idx] = (lp - lm) / (2 * eps)
        return num

    loss = lambda: _loss(w, X, hist_off, xt, tgt_off, dZ, dz, L_infer)
    for name in sorted(w):
        num = fd(loss, w[name])
        assert np.abs(num - G[name]).max() <= 1e-6 * max(1.0, np.abs(G[name]).max()), name
    num = fd(loss, X)
    assert np.abs(num - dX).max() <= 1e-6 * max(1.0, np.abs(dX).max())
    assert np.all(dX[4] == 0) and np.all(dX[3] == 0)  # dropped by the suffix / request without targets
    num = fd(loss, xt)
    assert np.abs(num - dxt).max() <= 1e-6 * max(1.0, np.abs(dxt).max())


def test_forward_pass_is_the_oracle_forward():
    w, X, hist_off, xt, tgt_off, dZ, dz = _case(1)
    _, _, _, Z, z = sb.backward(w, d=D, h=H, r=R, M=M, X=X, hist_off=hist_off, xt=xt, tgt_off=tgt_off,
                                dZ=dZ, dz=dz, L_infer=0)
    Zr, zr = oracle.forward(w, d=D, h=H, r=R, M=M, X=X, hist_off=hist_off, xt=xt, tgt_off=tgt_off,
                            L_infer=0, with_z=True, form=0)
    assert np.abs(Z - Zr).max() <= 1e-12 and np.abs(z - zr).max() <= 1e-12


def test_request_level_aggregation():
    """m targets sharing one history == m single-target requests over copies of it, gradients summed."""
    rng = np.random.default_rng(2)
    w = _weights(rng)
    L, m = 6, 3
    X = rng.standard_normal((L, D))
    xt = rng.standard_normal((m, D))
    dZ = rng.standard_normal((m, M, D))
    dz = rng.standard_normal((m, D))
    G1, dX1, dxt1, _, _ = sb.backward(w, d=D, h=H, r=R, M=M, X=X, hist_off=[0, L], xt=xt, tgt_off=[0, m],
                                      dZ=dZ, dz=dz)
    Gm, dXm, dxtm, _, _ = sb.backward(w, d=D, h=H, r=R, M=M, X=np.tile(X, (m, 1)),
                                      hist_off=np.arange(m + 1) * L, xt=xt, tgt_off=np.arange(m + 1),
                                      dZ=dZ, dz=dz)
    for k in G1:
        assert np.allclose(G1[k], Gm[k], rtol=1e-12, atol=1e-12), k
    assert np.allclose(dX1, dXm.reshape(m, L, D).sum(0), rtol=1e-12, atol=1e-12)
    assert np.allclose(dxt1, dxtm, rtol=1e-12, atol=1e-12)
