"""Pins for the f64 oracle (``oracle/``) against what the paper and the mathematics fix.

Every test here pins the oracle to something other than itself: a value printed
by the paper / SPEC worked examples (tests/golden/closed_forms.json), a closed
form, a special case that reduces to a textbook or library routine (torch's
multi-head attention / layer_norm / softmax / silu), an exact invariant stated by
the paper, or brute force on tiny inputs.  DESIGN.md "Oracle pins" maps each pin
to the paper passage (P1-P19 of SURVEY.md §8(c)).
"""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import workload

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))
RNG = np.random.default_rng(1234)


def rnd(*shape, scale=1.0):
    return RNG.standard_normal(shape) * scale


def uni(rows, cols):
    a = 1.0 / math.sqrt(rows)
    return RNG.uniform(-a, a, size=(rows, cols))


# --------------------------------------------------------------------------- P1
def test_swiglu_closed_forms():
    g = GOLD["swiglu_identity"]
    I = np.eye(2)
    out = oracle.swigluffn(np.array(g["x"]), I, I, I)[0]
    np.testing.assert_allclose(out, g["expected"], rtol=0, atol=1e-15)
    d, rd = 8, 32
    Wu, Wv, Wo = uni(d, rd), uni(d, rd), uni(rd, d)
    assert np.all(oracle.swigluffn(np.zeros((3, d)), Wu, Wv, Wo) == 0.0)
    x = rnd(5, d)
    np.testing.assert_allclose(oracle.swigluffn(x, Wu, Wv, 3.0 * Wo), 3.0 * oracle.swigluffn(x, Wu, Wv, Wo),
                               rtol=1e-14, atol=1e-15)


def test_swiglu_library():
    """Eq.(1) printed form: (x Wu) * silu(x Wv), then Wo -- torch.nn.functional.silu."""
    d, rd = 16, 64
    Wu, Wv, Wo = uni(d, rd), uni(d, rd), uni(rd, d)
    x = rnd(7, d)
    tx = torch.from_numpy(x)
    ref = ((tx @ torch.from_numpy(Wu)) * F.silu(tx @ torch.from_numpy(Wv))) @ torch.from_numpy(Wo)
    np.testing.assert_allclose(oracle.swigluffn(x, Wu, Wv, Wo), ref.numpy(), rtol=1e-12, atol=1e-13)
    # the gate is on Wv, not Wu: swapping must change the value (mutation sensitivity)
    assert np.abs(oracle.swigluffn(x, Wv, Wu, Wo) - ref.numpy()).max() > 1e-3


# --------------------------------------------------------------------------- P2
def test_layernorm_closed_forms_and_library():
    g = GOLD["layernorm_1_3"]
    np.testing.assert_allclose(oracle.layernorm(np.array(g["x"]), eps=g["eps"])[0], g["expected"], rtol=1e-15)
    beta = rnd(6)
    out = oracle.layernorm(np.full((2, 6), 3.25), g=rnd(6), b=beta)
    np.testing.assert_allclose(out, np.stack([beta, beta]), rtol=0, atol=1e-15)
    x, gg, bb = rnd(9, 24), rnd(24), rnd(24)
    ref = F.layer_norm(torch.from_numpy(x), (24,), torch.from_numpy(gg), torch.from_numpy(bb), eps=1e-5)
    np.testing.assert_allclose(oracle.layernorm(x, gg, bb), ref.numpy(), rtol=1e-12, atol=1e-13)


# --------------------------------------------------------------------------- P3
def test_softmax_closed_forms_and_library():
    g = GOLD["softmax_ln3"]
    np.testing.assert_allclose(oracle.softmax(np.array(g["logits"])), g["expected"], rtol=1e-15)
    np.testing.assert_allclose(oracle.softmax(np.full(7, 2.5)), np.full(7, 1 / 7), rtol=1e-15)
    s = rnd(50, scale=5)
    np.testing.assert_allclose(oracle.softmax(s + 123.0), oracle.softmax(s), rtol=1e-12)
    np.testing.assert_allclose(oracle.softmax(s), torch.softmax(torch.from_numpy(s), 0).numpy(), rtol=1e-13)


# --------------------------------------------------------------------------- layer fixtures
def layer_weights(d):
    return {k: uni(d, d) for k in ("WQ", "WK", "WV", "WO")}


def torch_mha(q, Xt, h, W):
    """Eq.(4)-(6) via torch's multi_head_attention_forward (query length 1, no biases).

    Row-vector convention x W  <->  torch's  W^T x, so in_proj = [WQ^T; WK^T; WV^T], out = WO^T;
    torch scales by 1/sqrt(d/h) = 1/sqrt(d_h) as Eq.(4) does.
    """
    d = q.shape[0]
    tq = torch.from_numpy(q).reshape(1, 1, d)
    tk = torch.from_numpy(Xt).reshape(-1, 1, d)
    in_w = torch.from_numpy(np.concatenate([W["WQ"].T, W["WK"].T, W["WV"].T], 0))
    out, _ = F.multi_head_attention_forward(
        tq, tk, tk, d, h, in_w, None, None, None, False, 0.0, torch.from_numpy(W["WO"].T), None,
        training=False, need_weights=False)
    return out.reshape(d).numpy()


# --------------------------------------------------------------------------- P19 (library routine)
@pytest.mark.parametrize("d,h,L", [(32, 1, 40), (64, 4, 300), (128, 4, 257)])
def test_attention_equals_torch_mha(d, h, L):
    W = layer_weights(d)
    q, Xt = rnd(d), rnd(L, d)
    ref = torch_mha(q, Xt, h, W)
    for form in (0, 1):
        np.testing.assert_allclose(oracle.attention(q, Xt, h, **W, form=form), ref, rtol=1e-11, atol=1e-12)


# --------------------------------------------------------------------------- P4, P5, P6
def test_single_key_alpha_is_one():
    d, h = 64, 4
    W = layer_weights(d)
    x1 = rnd(1, d)
    expected = x1[0] @ W["WV"] @ W["WO"]   # concat_r(x W_V^r) = x W_V  (closed form)
    for q in (rnd(d), rnd(d, scale=30)):
        for form in (0, 1):
            np.testing.assert_allclose(oracle.attention(q, x1, h, **W, form=form), expected, rtol=1e-13, atol=1e-14)


def test_identical_rows_equal_single_row():
    d, h = 32, 2
    W = layer_weights(d)
    x1 = rnd(1, d)
    q = rnd(d, scale=4)
    np.testing.assert_allclose(oracle.attention(q, np.repeat(x1, 37, 0), h, **W),
                               oracle.attention(q, x1, h, **W), rtol=1e-13, atol=1e-14)


def test_zero_query_weights_is_mean_pooling():
    d, h, L = 48, 3, 91
    W = layer_weights(d)
    W["WQ"] = np.zeros((d, d))
    Xt = rnd(L, d)
    expected = Xt.mean(0) @ W["WV"] @ W["WO"]
    np.testing.assert_allclose(oracle.attention(rnd(d), Xt, h, **W), expected, rtol=1e-12, atol=1e-13)


# --------------------------------------------------------------------------- full-forward fixtures
def small_workload(seed=0, B=3, m=2, d=32, h=4, M=3, lengths=None, shared=True, L_infer=0, ln_affine=True):
    cfg = workload.Config("pin", B=B, m=m, d=d, h=h, r=2, M=M, dtype="fp32", L_fixed=16,
                          shared_ffn=shared, L_infer=L_infer)
    if lengths is None:
        lengths = np.array([5, 17, 1] + [9] * (B - 3))[:B]
    return workload.make_workload(cfg, seed=seed, lengths=lengths, ln_affine=ln_affine)


def run(wl, **kw):
    Z, z, _ = oracle.forward_workload(wl, **kw)
    return Z, z


# --------------------------------------------------------------------------- P16 brute force / library model
def torch_stack(wl):
    """The stack of PAPER.md §3.1 written directly from Eq.(1)-(9) with torch library routines
    (F.silu, F.layer_norm, F.multi_head_attention_forward), independent of the oracle's code."""
    c = wl.cfg
    W = {k: torch.from_numpy(np.asarray(v, dtype=np.float64)) for k, v in workload.full_weights(wl).items()}
    d, h, M = c.d, c.h, c.M

    def ffn(x, p):
        return ((x @ W[p + ".Wu"]) * F.silu(x @ W[p + ".Wv"])) @ W[p + ".Wo"]

    def ln(x, p):
        return F.layer_norm(x, (d,), W[p + ".ln_g"].reshape(d), W[p + ".ln_b"].reshape(d), eps=1e-5)

    X = torch.from_numpy(wl.X.astype(np.float64))
    xt = torch.from_numpy(wl.xt.astype(np.float64))
    Z = torch.zeros(wl.Nt, M, d, dtype=torch.float64)
    zz = torch.zeros(wl.Nt, d, dtype=torch.float64)
    for b in range(len(wl.lengths)):
        s, e = int(wl.hist_off[b]), int(wl.hist_off[b + 1])
        if c.L_infer:
            s = max(s, e - c.L_infer)
        Xb = X[s:e]
        Xts = [ln(ffn(Xb, f"L{i}.hist"), f"L{i}.hist") for i in range(1, M + 1)]
        for t in range(int(wl.tgt_off[b]), int(wl.tgt_off[b + 1])):
            q = ln(ffn(xt[t], "L1.qry"), "L1.qry")
            os_ = []
            for i in range(1, M + 1):
                Wl = {k: W[f"L{i}.{k}"].numpy() for k in ("WQ", "WK", "WV", "WO")}
                o = torch.from_numpy(torch_mha(q.numpy(), Xts[i - 1].numpy(), h, Wl))
                os_.append(o)
                Z[t, i - 1] = o
                if i < M:
                    q = ffn(torch.cat(os_ + [xt[t]]) @ W[f"L{i + 1}.WC"], f"L{i + 1}.qry")
            zz[t] = ffn(torch.cat(os_ + [xt[t]]) @ W["z.WZ"], "z")
    return Z.numpy(), zz.numpy()


@pytest.mark.parametrize("shared", [True, False])
def test_full_stack_equals_library_model(shared):
    wl = small_workload(shared=shared)
    Zr, zr = torch_stack(wl)
    for form in (0, 1):
        Z, z = run(wl, form=form)
        np.testing.assert_allclose(Z, Zr, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(z, zr, rtol=1e-10, atol=1e-12)


def test_tiny_config_equals_library_model():
    wl = workload.make_workload("tiny", seed=3)
    Zr, zr = torch_stack(wl)
    Z, z = run(wl)
    np.testing.assert_allclose(Z, Zr, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(z, zr, rtol=1e-10, atol=1e-12)


# --------------------------------------------------------------------------- P8 dual form
def test_standard_equals_reordered_full_stack():
    wl = small_workload(B=4, m=3, d=64, h=4, M=4, lengths=np.array([200, 3, 64, 129]))
    Z0, z0 = run(wl, form=0)
    Z1, z1 = run(wl, form=1)
    rel = np.abs(Z0 - Z1).max(-1) / np.abs(Z0).max(-1)
    assert rel.max() < 1e-12
    assert (np.abs(z0 - z1).max(-1) / np.abs(z0).max(-1)).max() < 1e-12


# --------------------------------------------------------------------------- P10 RLB
def test_rlb_batched_equals_independent_bit_exact():
    """RLB: m targets sharing one history == m single-target requests."""
    wl = small_workload(B=2, m=4, lengths=np.array([23, 11]))
    Z, z = run(wl)
    for b in range(2):
        s, e = wl.hist_off[b], wl.hist_off[b + 1]
        for t in range(wl.tgt_off[b], wl.tgt_off[b + 1]):
            Z1, z1 = oracle.forward(workload.full_weights(wl), d=wl.cfg.d, h=wl.cfg.h, r=wl.cfg.r, M=wl.cfg.M,
                                    X=wl.X[s:e], hist_off=[0, e - s], xt=wl.xt[t:t + 1], tgt_off=[0, 1])
            assert np.array_equal(Z1[0], Z[t]) and np.array_equal(z1[0], z[t])


# --------------------------------------------------------------------------- P9 ragged layout
def test_ragged_segments_independent_and_permutation_equivariant():
    wl = small_workload(B=4, m=2, lengths=np.array([7, 30, 2, 12]))
    Z, z = run(wl)
    perm = [2, 0, 3, 1]
    Zp, zp, rows = oracle.forward_workload(wl, requests=perm)
    assert np.array_equal(Zp, Z[rows]) and np.array_equal(zp, z[rows])
    # perturbing request 1's history leaves every other request's outputs bit-identical
    X2 = wl.X.copy()
    X2[wl.hist_off[1]:wl.hist_off[2]] += 0.5
    Z2, _ = oracle.forward(workload.full_weights(wl), d=wl.cfg.d, h=wl.cfg.h, r=wl.cfg.r, M=wl.cfg.M, X=X2,
                           hist_off=wl.hist_off, xt=wl.xt, tgt_off=wl.tgt_off)
    other = np.r_[0:2, 4:8]
    assert np.array_equal(Z2[other], Z[other]) and not np.array_equal(Z2[2:4], Z[2:4])


def test_ragged_equals_padded_masked():
    """Ragged Target Attention == pad-to-max + -inf mask, via torch MHA's key_padding_mask."""
    d, h = 32, 4
    W = layer_weights(d)
    lengths = [3, 11, 6]
    Lmax = max(lengths)
    Xs = [rnd(L, d) for L in lengths]
    q = rnd(3, d)
    pad = np.zeros((Lmax, 3, d))
    mask = np.ones((3, Lmax), dtype=bool)
    for b, L in enumerate(lengths):
        pad[:L, b] = Xs[b]
        mask[b, :L] = False
    in_w = torch.from_numpy(np.concatenate([W["WQ"].T, W["WK"].T, W["WV"].T], 0))
    out, _ = F.multi_head_attention_forward(
        torch.from_numpy(q).reshape(1, 3, d), torch.from_numpy(pad), torch.from_numpy(pad), d, h, in_w, None,
        None, None, False, 0.0, torch.from_numpy(W["WO"].T), None, training=False,
        key_padding_mask=torch.from_numpy(mask), need_weights=False)
    for b in range(3):
        np.testing.assert_allclose(oracle.attention(q[b], Xs[b], h, **W), out[0, b].numpy(), rtol=1e-11, atol=1e-12)


# --------------------------------------------------------------------------- P7, P12 invariants
def test_history_duplication_and_permutation_invariance():
    wl = small_workload(B=1, m=3, lengths=np.array([40]))
    Z, z = run(wl)
    W = workload.full_weights(wl)
    c = wl.cfg
    kw = dict(d=c.d, h=c.h, r=c.r, M=c.M, xt=wl.xt, tgt_off=wl.tgt_off)
    Zd, zd = oracle.forward(W, X=np.concatenate([wl.X, wl.X]), hist_off=[0, 80], **kw)
    np.testing.assert_allclose(Zd, Z, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(zd, z, rtol=1e-12, atol=1e-13)
    perm = np.random.default_rng(5).permutation(40)
    Zp, zp = oracle.forward(W, X=wl.X[perm], hist_off=[0, 40], **kw)
    np.testing.assert_allclose(Zp, Z, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(zp, z, rtol=1e-12, atol=1e-13)


# --------------------------------------------------------------------------- P11 fusion selector
def test_fusion_selector_reduces_to_ffn_of_o1():
    """Eq.(7) with W_C(2) = [I; 0] -> q(2) = SwiGLUFFN(2)(o(1))."""
    wl = small_workload(B=1, m=2, M=2, lengths=np.array([19]))
    d = wl.cfg.d
    wl.weights["L2.WC"] = np.concatenate([np.eye(d), np.zeros((d, d))]).astype(np.float32)
    W = workload.full_weights(wl)
    Z, _ = run(wl)
    Xt2 = F.layer_norm(torch.from_numpy(oracle.swigluffn(wl.X, W["L2.hist.Wu"], W["L2.hist.Wv"], W["L2.hist.Wo"])),
                       (d,), torch.from_numpy(W["L2.hist.ln_g"].reshape(d).astype(np.float64)),
                       torch.from_numpy(W["L2.hist.ln_b"].reshape(d).astype(np.float64)), eps=1e-5).numpy()
    Wl = {k: W["L2." + k].astype(np.float64) for k in ("WQ", "WK", "WV", "WO")}
    for t in range(2):
        q2 = oracle.swigluffn(Z[t, 0], W["L2.qry.Wu"], W["L2.qry.Wv"], W["L2.qry.Wo"])[0]
        np.testing.assert_allclose(Z[t, 1], torch_mha(q2, Xt2, wl.cfg.h, Wl), rtol=1e-10, atol=1e-12)
    # all-zero inputs propagate to a zero query: zero x_t and zero W_O -> q(2) = 0
    assert np.all(oracle.swigluffn(np.zeros(d) @ W["L2.WC"][:d], W["L2.qry.Wu"], W["L2.qry.Wv"], W["L2.qry.Wo"]) == 0)


# --------------------------------------------------------------------------- P13, P14 suffix / length agnosticism
def test_suffix_golden():
    g = GOLD["suffix_examples"]
    assert oracle.suffix_starts(g["hist_off"], g["L_infer"]).tolist() == g["expected_start"]


def test_L_infer_equals_explicit_slice_bit_exact():
    wl = small_workload(B=3, m=2, lengths=np.array([50, 9, 33]), L_infer=20)
    Z, z = run(wl)
    W = workload.full_weights(wl)
    for b in range(3):
        s, e = wl.hist_off[b], wl.hist_off[b + 1]
        s2 = max(s, e - 20)
        t0, t1 = wl.tgt_off[b], wl.tgt_off[b + 1]
        Zb, zb = oracle.forward(W, d=wl.cfg.d, h=wl.cfg.h, r=wl.cfg.r, M=wl.cfg.M, X=wl.X[s2:e],
                                hist_off=[0, e - s2], xt=wl.xt[t0:t1], tgt_off=[0, t1 - t0])
        assert np.array_equal(Zb, Z[t0:t1]) and np.array_equal(zb, z[t0:t1])
    # cap >= every length is the identity
    Zn, _ = run(wl, L_infer=0)
    Zc, _ = run(wl, L_infer=50)
    assert np.array_equal(Zn, Zc)


def test_length_agnostic_shapes():
    for L in (16, 1000):
        wl = small_workload(B=1, m=2, lengths=np.array([L]))
        Z, z = run(wl)
        assert Z.shape == (2, wl.cfg.M, wl.cfg.d) and z.shape == (2, wl.cfg.d) and np.isfinite(Z).all()


# --------------------------------------------------------------------------- validation
def test_validation_errors():
    wl = small_workload()
    W = workload.full_weights(wl)
    c = wl.cfg
    kw = dict(d=c.d, h=c.h, r=c.r, M=c.M, xt=wl.xt)
    with pytest.raises(oracle.OracleError) as e:
        oracle.forward(W, X=wl.X, hist_off=[0, 5, 5, 23], tgt_off=[0, 2, 4, 6], **kw)
    assert e.value.status == oracle.ERR_EMPTY_HISTORY and e.value.index == 1
    with pytest.raises(oracle.OracleError) as e:
        oracle.forward(W, X=wl.X, hist_off=[0, 5, 4, 23], tgt_off=[0, 2, 4, 6], **kw)
    assert e.value.status == oracle.ERR_OFFSETS
    with pytest.raises(oracle.OracleError) as e:
        oracle.forward(W, X=wl.X, hist_off=[0, 5, 10, 20], tgt_off=[0, 2, 4, 6], **kw)
    assert e.value.status == oracle.ERR_OFFSETS
    # m_b = 0 is legal
    Z, _ = oracle.forward(W, X=wl.X, hist_off=wl.hist_off, tgt_off=[0, 0, 3, 6], **kw)
    assert Z.shape[0] == 6


# --------------------------------------------------------------------------- generator facts (Eq.16-17)
def test_beta_and_reduction_factor_golden():
    g = GOLD["beta_shape"]
    assert workload.beta_for(g["alpha"], g["L_min"], g["L_max"], g["L_avg"]) == pytest.approx(g["expected"], rel=1e-15)
    g = GOLD["reorder_reduction_factor"]
    assert 2 * (g["d"] // g["h"]) == g["expected"]


def test_length_sampler_mean_and_rounding():
    cfg = workload.CONFIGS["train"]
    L = workload.sample_lengths(np.random.default_rng(0), cfg, 20000)
    assert np.all(L % 8 == 0) and L.min() >= 8 and L.max() <= cfg.L_max
    assert abs(L.mean() - cfg.L_avg) / cfg.L_avg < 0.03   # E[L_raw] = L_avg by Eq.(17)
