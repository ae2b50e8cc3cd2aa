"""Oracle of the backward of the WHOLE STCA stack under RLB -- TEST INFRASTRUCTURE ONLY.

Only tests/ may import this module; the product path (paper_2511_06077_b200/) never does.  Plain numpy,
float64, one request at a time (vectorised over its targets), every step written out in the order of
the forward it differentiates:

    Eq.(2)  X~(i) = LN_H(i)(SwiGLUFFN_H(i)(X))                     P:L111   (from raw X per layer, R4)
    Eq.(3)  q(1)  = LN_Q(1)(SwiGLUFFN_Q(1)(x_t))
    Eq.(4)  alpha(i,r) = softmax(q W_Q^r (X~ W_K^r)^T / sqrt(d_h))  P:L122-125  (standard form, Eq.(12))
    Eq.(5)  o(i,r) = alpha (X~ W_V^r)
    Eq.(6)  o(i) = [o(i,1) | ... | o(i,h)] W_O
    Eq.(7)  q(i+1) = SwiGLUFFN_Q(i+1)([o(1) | ... | o(i) | x_t] W_C(i+1))   P:L138-141  (x_t last, R10)
    Eq.(8)  Z_H = [o(1); ...; o(M)]
    Eq.(9)  z = SwiGLUFFN_Z([o(1) | ... | o(M) | x_t] W_Z)

with SwiGLUFFN(x) = ((x Wu) * silu(x Wv)) Wo (Eq.(1); R1-R3: no biases, biased variance,
eps inside the root).  The loss is the vector-Jacobian product with given upstream gradients,

    loss = sum(dZ * Z_H) + sum(dz * z),

so the result is (d loss / d every weight role, d loss / d X, d loss / d x_t).  The RLB property
(P:L205-210): the history path of a request -- X~(i) and its K/V -- is computed once and
shared by all m_b targets, so its gradients are summed over the request's targets here, inside the
request, before anything is added across requests.  History rows a request drops by the L_infer
suffix take no part in the forward and get a zero gradient.

Gradients are per ROLE name (the names of include/stca.h's weights).  Where one parameter serves
several roles (the shared-FFN reading R5 passes the history FFN of layer i as its query FFN too), its
gradient is the sum of its roles' gradients.

Pinned in tests/test_oracle_stack_backward.py by central finite differences of the C oracle's forward
(oracle.forward, a separate code path, standard form) over every weight entry and input of a tiny
stack, by the oracle forward itself (this module's forward pass must reproduce oracle.forward), and by
the request-level aggregation identity.
"""
from __future__ import annotations

from typing import Dict

import numpy as np


def _sig(g):
    return 1.0 / (1.0 + np.exp(-g))


def _ffn(x, Wu, Wv, Wo):
    """Eq.(1) with its cache."""
    a, g = x @ Wu, x @ Wv
    s = _sig(g)
    H = a * g * s
    return H @ Wo, (x, a, g, s, H)


def _ffn_bwd(dy, cache, Wu, Wv, Wo):
    """(dx, dWu, dWv, dWo) of Eq.(1): silu'(g) = s (1 + g (1 - s))."""
    x, a, g, s, H = cache
    dWo = H.T @ dy
    dH = dy @ Wo.T
    da = dH * g * s
    dg = dH * a * s * (1.0 + g * (1.0 - s))
    return da @ Wu.T + dg @ Wv.T, x.T @ da, x.T @ dg, dWo


def _ln(y, gam, bet, eps):
    mu = y.mean(1, keepdims=True)
    sd = np.sqrt(((y - mu) ** 2).mean(1, keepdims=True) + eps)
    xh = (y - mu) / sd
    return xh * gam + bet, (xh, sd)


def _ln_bwd(dout, cache, gam):
    """(dy, dgamma, dbeta) of the LayerNorm."""
    xh, sd = cache
    dxh = dout * gam
    dy = (dxh - dxh.mean(1, keepdims=True) - xh * (dxh * xh).mean(1, keepdims=True)) / sd
    return dy, (dout * xh).sum(0), dout.sum(0)


def _softmax(S):
    P = np.exp(S - S.max(1, keepdims=True))
    return P / P.sum(1, keepdims=True)


def backward(weights: Dict[str, np.ndarray], *, d: int, h: int, r: int, M: int, X, hist_off, xt, tgt_off,
             dZ, dz=None, L_infer: int = 0, ln_eps: float = 1e-5, with_z: bool = True):
    """Returns (grads: role -> array shaped like the weight, dX [T x d], dxt [Nt x d], Z [Nt x M x d], z)."""
    W = {k: np.asarray(v, np.float64).reshape(v.shape if np.ndim(v) == 2 else (1, -1)) for k, v in weights.items()}
    X, xt = np.asarray(X, np.float64).reshape(-1, d), np.asarray(xt, np.float64).reshape(-1, d)
    dZ = np.asarray(dZ, np.float64).reshape(-1, M, d)
    hist_off, tgt_off = np.asarray(hist_off, np.int64), np.asarray(tgt_off, np.int64)
    B = len(hist_off) - 1
    dh = d // h
    isq = 1.0 / np.sqrt(dh)
    G = {k: np.zeros_like(v) for k, v in W.items()}
    dX, dxt = np.zeros_like(X), np.zeros_like(xt)
    Z = np.zeros((xt.shape[0], M, d))
    z = np.zeros((xt.shape[0], d)) if with_z else None
    vec = lambda a: a.reshape(-1)  # ln_g / ln_b are [1 x d]

    for b in range(B):
        t0, t1 = int(tgt_off[b]), int(tgt_off[b + 1])
        if t1 == t0:
            continue  # no targets: no output depends on this request
        e0 = int(hist_off[b + 1])
        s0 = max(int(hist_off[b]), e0 - L_infer) if L_infer > 0 else int(hist_off[b])  # temporal suffix
        Xb, xb = X[s0:e0], xt[t0:t1]
        m = t1 - t0
        # ---------------- forward, caching what the backward needs ----------------
        hc, lc, Xt = [None] * (M + 1), [None] * (M + 1), [None] * (M + 1)
        for i in range(1, M + 1):  # Eq.(2): once per request (RLB)
            p = f"L{i}.hist."
            y, hc[i] = _ffn(Xb, W[p + "Wu"], W[p + "Wv"], W[p + "Wo"])
            Xt[i], lc[i] = _ln(y, vec(W[p + "ln_g"]), vec(W[p + "ln_b"]), ln_eps)
        q, qc, cin = [None] * (M + 1), [None] * (M + 1), [None] * (M + 1)
        y1, qc[1] = _ffn(xb, W["L1.qry.Wu"], W["L1.qry.Wv"], W["L1.qry.Wo"])  # Eq.(3)
        q[1], q1ln = _ln(y1, vec(W["L1.qry.ln_g"]), vec(W["L1.qry.ln_b"]), ln_eps)
        o, att = [None] * (M + 1), [None] * (M + 1)
        for i in range(1, M + 1):
            p = f"L{i}."
            cat = np.zeros((m, d))
            heads = []
            for hr in range(h):  # Eq.(4)-(5), head r = columns [r d_h, (r+1) d_h)
                C = slice(hr * dh, (hr + 1) * dh)
                qh = q[i] @ W[p + "WQ"][:, C]
                K, V = Xt[i] @ W[p + "WK"][:, C], Xt[i] @ W[p + "WV"][:, C]
                A = _softmax(qh @ K.T * isq)
                cat[:, C] = A @ V
                heads.append((qh, K, V, A))
            o[i] = cat @ W[p + "WO"]  # Eq.(6)
            att[i] = (cat, heads)
            Z[t0:t1, i - 1] = o[i]  # Eq.(8)
            if i < M:  # Eq.(7)
                pn = f"L{i + 1}."
                cin[i + 1] = np.concatenate(o[1:i + 1] + [xb], axis=1)
                q[i + 1], qc[i + 1] = _ffn(cin[i + 1] @ W[pn + "WC"], W[pn + "qry.Wu"], W[pn + "qry.Wv"],
                                           W[pn + "qry.Wo"])
        # ---------------- backward ----------------
        do = [None] + [dZ[t0:t1, i - 1].copy() for i in range(1, M + 1)]
        dxb = np.zeros_like(xb)
        if with_z:  # Eq.(9)
            zin = np.concatenate(o[1:M + 1] + [xb], axis=1)
            zc_in = zin @ W["z.WZ"]
            z[t0:t1], zc = _ffn(zc_in, W["z.Wu"], W["z.Wv"], W["z.Wo"])
            if dz is not None:
                dzb = np.asarray(dz, np.float64).reshape(-1, d)[t0:t1]
                dc, gu, gv, go = _ffn_bwd(dzb, zc, W["z.Wu"], W["z.Wv"], W["z.Wo"])
                G["z.Wu"] += gu
                G["z.Wv"] += gv
                G["z.Wo"] += go
                G["z.WZ"] += zin.T @ dc
                dzin = dc @ W["z.WZ"].T
                for j in range(1, M + 1):
                    do[j] += dzin[:, (j - 1) * d:j * d]
                dxb += dzin[:, M * d:]
        for i in range(M, 0, -1):  # do[i] is complete: layers > i have added their W_C terms
            p = f"L{i}."
            cat, heads = att[i]
            G[p + "WO"] += cat.T @ do[i]
            dcat = do[i] @ W[p + "WO"].T
            dq = np.zeros((m, d))
            dXt = np.zeros_like(Xt[i])
            for hr, (qh, K, V, A) in enumerate(heads):
                C = slice(hr * dh, (hr + 1) * dh)
                dc_r = dcat[:, C]
                dV = A.T @ dc_r
                dA = dc_r @ V.T
                dS = A * (dA - (dA * A).sum(1, keepdims=True)) * isq
                dqh, dK = dS @ K, dS.T @ qh  # dK sums over ALL the request's targets (RLB)
                G[p + "WQ"][:, C] += q[i].T @ dqh
                G[p + "WK"][:, C] += Xt[i].T @ dK
                G[p + "WV"][:, C] += Xt[i].T @ dV
                dq += dqh @ W[p + "WQ"][:, C].T
                dXt += dK @ W[p + "WK"][:, C].T + dV @ W[p + "WV"][:, C].T
            # history path of layer i (Eq.(2))
            dy, gg, gb = _ln_bwd(dXt, lc[i], vec(W[p + "hist.ln_g"]))
            G[p + "hist.ln_g"] += gg.reshape(G[p + "hist.ln_g"].shape)
            G[p + "hist.ln_b"] += gb.reshape(G[p + "hist.ln_b"].shape)
            dXh, gu, gv, go = _ffn_bwd(dy, hc[i], W[p + "hist.Wu"], W[p + "hist.Wv"], W[p + "hist.Wo"])
            G[p + "hist.Wu"] += gu
            G[p + "hist.Wv"] += gv
            G[p + "hist.Wo"] += go
            dX[s0:e0] += dXh
            # query path of layer i
            if i >= 2:  # Eq.(7)
                dc, gu, gv, go = _ffn_bwd(dq, qc[i], W[p + "qry.Wu"], W[p + "qry.Wv"], W[p + "qry.Wo"])
                G[p + "qry.Wu"] += gu
                G[p + "qry.Wv"] += gv
                G[p + "qry.Wo"] += go
                G[p + "WC"] += cin[i].T @ dc
                dcin = dc @ W[p + "WC"].T
                for j in range(1, i):
                    do[j] += dcin[:, (j - 1) * d:j * d]
                dxb += dcin[:, (i - 1) * d:]
            else:  # Eq.(3)
                dy1, gg, gb = _ln_bwd(dq, q1ln, vec(W["L1.qry.ln_g"]))
                G["L1.qry.ln_g"] += gg.reshape(G["L1.qry.ln_g"].shape)
                G["L1.qry.ln_b"] += gb.reshape(G["L1.qry.ln_b"].shape)
                dx1, gu, gv, go = _ffn_bwd(dy1, qc[1], W["L1.qry.Wu"], W["L1.qry.Wv"], W["L1.qry.Wo"])
                G["L1.qry.Wu"] += gu
                G["L1.qry.Wv"] += gv
                G["L1.qry.Wo"] += go
                dxb += dx1
        dxt[t0:t1] = dxb
    return G, dX, dxt, Z, z
