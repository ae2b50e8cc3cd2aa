"""Oracle of the attention backward with request-level gradient aggregation (SURVEY §8(f) NEXT-1,
partial) -- TEST INFRASTRUCTURE ONLY.

Only tests/ may import this module; the product path (paper_2511_06077_b200/) never does.  Plain
numpy, float64, one request at a time, the textbook softmax-attention backward written out.

What it differentiates.  One layer's ragged single-query attention in the reordered form the GPU
runs (Eq.(13)): for request b with history rows X~_b [L_b x d] and query rows U_b
[m_b h x d] (the reordered queries u = q W_QK, already scaled by log2(e)/sqrt(d_h), so the scores are
in the log2 domain),

    S = U_b X~_b^T,   alpha = 2^S / rowsum(2^S)  (= softmax(ln 2 * S)),   Y_b = alpha X~_b.

Given dY_b = dLoss/dY_b:

    D    = rowsum(dY_b * Y_b)                         [m_b h]
    dS   = ln 2 * alpha * (dY_b X~_b^T - D)          [m_b h x L_b]
    dX~_b = alpha^T dY_b + dS^T U_b                    [L_b x d]
    dU_b = dS X~_b                                     [m_b h x d]

dX~_b sums over ALL of the request's query rows (its m_b targets x h heads): the gradient of the
shared history encoding is aggregated at the request level before anything leaves the request --
the RLB property of P:L396 ("aggregate gradients at the request level before synchronization") and
P:L219 (the K/V-like activations are shared by the m targets).  Pinned in
tests/test_oracle_attention_backward.py by central finite differences of the forward below (a
separate code path), closed forms (one history row; zero queries) and the aggregation identity.
"""
from __future__ import annotations

import numpy as np

LN2 = float(np.log(2.0))


def forward(U, Xt, hist_len, q_off):
    """Y [NQ x d]: per request b, alpha = softmax over its keys of 2^(U X~^T), Y = alpha X~."""
    U, Xt = np.asarray(U, np.float64), np.asarray(Xt, np.float64)
    Y = np.zeros_like(U)
    k0 = 0
    for b in range(len(hist_len)):
        Xb = Xt[k0:k0 + hist_len[b]]
        k0 += hist_len[b]
        for q in range(q_off[b], q_off[b + 1]):
            s = Xb @ U[q]
            p = np.exp2(s - s.max())
            Y[q] = (p / p.sum()) @ Xb
    return Y


def backward(U, Xt, dY, hist_len, q_off):
    """(dX~ [T' x d], dU [NQ x d]) of the layer above, requests back to back in cache order."""
    U, Xt, dY = (np.asarray(a, np.float64) for a in (U, Xt, dY))
    dX = np.zeros_like(Xt)
    dU = np.zeros_like(U)
    k0 = 0
    for b in range(len(hist_len)):
        Lb = hist_len[b]
        Xb = Xt[k0:k0 + Lb]
        q0, q1 = q_off[b], q_off[b + 1]
        if q1 > q0:
            S = U[q0:q1] @ Xb.T
            A = np.exp2(S - S.max(1, keepdims=True))
            A /= A.sum(1, keepdims=True)                  # alpha
            Yb = A @ Xb
            D = (dY[q0:q1] * Yb).sum(1, keepdims=True)
            dS = LN2 * A * (dY[q0:q1] @ Xb.T - D)
            dX[k0:k0 + Lb] = A.T @ dY[q0:q1] + dS.T @ U[q0:q1]
            dU[q0:q1] = dS @ Xb
        k0 += Lb
    return dX, dU
