"""Stage-isolated GPU checks (SURVEY §8(c) "stage-isolated tolerances", I4 output placement).

* The fused history projection alone (a1, Eq.(2)): the X~ cache read back through stca_read_cache
  against the f64 oracle's LN(SwiGLUFFN(X)) of the same bf16 X and weights, every row of every
  layer of a few ragged serve-shaped requests, row-inf-relative <= 1e-2 (bf16: G and X~ rounding,
  SURVEY measured 5.5-5.9e-3) and <= 1e-4 on the fp32 path.
* I4: permuting the targets inside each request permutes the output rows bit-exactly."""
import numpy as np
import pytest

import oracle
import workload
from _util import device_inputs, make_cfg, rowrel, run_gpu

pytestmark = pytest.mark.gpu


def _projected(wl, dtype):
    import torch
    import paper_2511_06077_b200 as stca
    c = wl.cfg
    m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=dtype)
    X, _ = device_inputs(wl)
    m.project_history(X, wl.hist_off)
    torch.cuda.synchronize()
    return m


@pytest.mark.parametrize("dtype,tol", [("bf16", 1e-2), ("fp32", 1e-4)])
def test_projection_cache_matches_oracle(dtype, tol):
    lengths = np.array([1000, 1, 333, 130, 2049])  # ragged: several 128-row tiles, an odd tile count
    cfg = make_cfg(B=len(lengths), m=2, dtype=dtype, M=4)
    wl = workload.make_workload(cfg, seed=11, lengths=lengths, ln_affine=True)
    m = _projected(wl, dtype)
    T = int(wl.hist_off[-1])
    w = wl.weights
    for i in range(1, cfg.M + 1):
        got = m.read_cache(i, 0, T)
        ref = oracle.layernorm(oracle.swigluffn(wl.X, w[f"L{i}.hist.Wu"], w[f"L{i}.hist.Wv"], w[f"L{i}.hist.Wo"]),
                               w[f"L{i}.hist.ln_g"], w[f"L{i}.hist.ln_b"])
        e = rowrel(got, ref)
        assert np.isfinite(got).all()
        assert e.max() <= tol, (i, e.max(), int(e.argmax()))


def test_projection_cache_suffix_order():
    """With L_infer the cache holds each request's LAST L_infer rows, requests back to back."""
    lengths = np.array([700, 90, 1500])
    cfg = make_cfg(B=3, m=2, L_infer=256)
    wl = workload.make_workload(cfg, seed=12, lengths=lengths)
    m = _projected(wl, "bf16")
    kept = np.minimum(lengths, 256)
    rows = np.concatenate([np.arange(wl.hist_off[b + 1] - kept[b], wl.hist_off[b + 1]) for b in range(3)])
    got = m.read_cache(2, 0, int(kept.sum()))
    w = wl.weights
    ref = oracle.layernorm(oracle.swigluffn(wl.X[rows], w["L2.hist.Wu"], w["L2.hist.Wv"], w["L2.hist.Wo"]),
                           w["L2.hist.ln_g"], w["L2.hist.ln_b"])
    assert rowrel(got, ref).max() <= 1e-2


def test_read_cache_errors():
    import paper_2511_06077_b200 as stca
    cfg = make_cfg(B=1, m=1, M=2)
    wl = workload.make_workload(cfg, seed=1, lengths=np.array([40]))
    c = wl.cfg
    m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M)
    with pytest.raises(stca.StcaError) as e:
        m.read_cache(1, 0, 4)
    assert e.value.status == -6
    X, _ = device_inputs(wl)
    m.project_history(X, wl.hist_off)
    for layer, r0, n in ((0, 0, 4), (3, 0, 4), (1, 38, 4)):
        with pytest.raises(stca.StcaError) as e:
            m.read_cache(layer, r0, n)
        assert e.value.status == -1


def test_target_permutation_permutes_outputs_bit_exact():
    """I4: permuting targets within each request permutes out_Z / out_z rows bit-exactly."""
    lengths = np.array([5000, 64, 900])
    cfg = make_cfg(B=3, m=48, L_infer=0)  # 48 targets x 4 heads = 192 query rows: a full and a partial tile
    wl = workload.make_workload(cfg, seed=13, lengths=lengths)
    Z, z = run_gpu(wl)
    rng = np.random.default_rng(0)
    perm = np.concatenate([wl.tgt_off[b] + rng.permutation(wl.tgt_off[b + 1] - wl.tgt_off[b]) for b in range(3)])
    wl2 = workload.Workload(cfg=wl.cfg, seed=wl.seed, weights=wl.weights, lengths=wl.lengths, hist_off=wl.hist_off,
                            tgt_off=wl.tgt_off, X=wl.X, xt=wl.xt[perm], X_bits=wl.X_bits, xt_bits=wl.xt_bits[perm])
    Zp, zp = run_gpu(wl2)
    assert np.array_equal(Zp, Z[perm]) and np.array_equal(zp, z[perm])


def test_degenerate_batches():
    """No targets at all (every m_b = 0): forward is a no-op on zero rows; a batch whose requests all
    have one history row and one target; repeated forwards on one projection are bit-identical."""
    import torch
    import paper_2511_06077_b200 as stca
    cfg = make_cfg(B=3, m=1, M=2)
    wl = workload.make_workload(cfg, seed=21, lengths=np.array([5, 1, 300]))
    c = wl.cfg
    m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M)
    X, xt = device_inputs(wl)
    m.project_history(X, wl.hist_off)
    Z0 = torch.zeros(0, c.M, c.d, device="cuda")
    m.forward(xt[:0], np.zeros(4, dtype=np.int64), Z0, torch.zeros(0, c.d, device="cuda"))
    torch.cuda.synchronize()
    Z1 = torch.full((wl.Nt, c.M, c.d), float("nan"), device="cuda")
    Z2 = torch.full((wl.Nt, c.M, c.d), float("nan"), device="cuda")
    m.forward(xt, wl.tgt_off, Z1)
    m.forward(xt, wl.tgt_off, Z2)
    torch.cuda.synchronize()
    assert torch.isfinite(Z1).all() and torch.equal(Z1, Z2)
    Zr, _, rows = oracle.forward_workload(wl, nthreads=2)
    assert rowrel(Z1.cpu().numpy()[rows], Zr).max() <= 2e-2
    wl1 = workload.make_workload(make_cfg(B=4, m=1, M=2), seed=22, lengths=np.ones(4, dtype=np.int64))
    Z, z = run_gpu(wl1)
    Zr, zr, rows = oracle.forward_workload(wl1, nthreads=2)
    assert rowrel(Z[rows], Zr).max() <= 2e-2 and rowrel(z[rows], zr).max() <= 2e-2


def _f64_attention(U, Xc, hist_len, tgt_off, h):
    """f64 reference of a4 on the GPU's own operands: for each query row u (log2 domain, pre-scaled by
    log2(e)/sqrt(d_h)) of request b, alpha = 2^(u X~_b^T) / sum, y = alpha X~_b (Eq.(13)).
    Also returns A = alpha |X~_b| (elementwise), the scale of every rounding error below."""
    Y = np.zeros_like(U)
    A = np.zeros_like(U)
    k0 = 0
    for b in range(len(hist_len)):
        Xb = Xc[k0:k0 + hist_len[b]]
        k0 += hist_len[b]
        q0, q1 = tgt_off[b] * h, tgt_off[b + 1] * h
        if q1 == q0:
            continue
        s = U[q0:q1] @ Xb.T
        p = np.exp2(s - s.max(1, keepdims=True))
        alpha = p / p.sum(1, keepdims=True)
        Y[q0:q1] = alpha @ Xb
        A[q0:q1] = alpha @ np.abs(Xb)
    return Y, A


# K-C stage bound, derived from the kernel's arithmetic: y_gpu = sum_j bf16(p_j) x_j / l
# with the sum l of the unrounded fp32 p_j, so rounding P to bf16 (relative 2^-9 per weight) moves y_e
# by at most 2^-9 A_e, A_e = sum_j alpha_j |x_je|; a split-K partial is stored as bf16(O/l) (another
# 2^-9 A_e after the fold's convex combination) and Y itself is rounded to bf16 (2^-9 |y_e| <= 2^-9 A_e);
# the exponentials (MUFU ex2.approx and the FMA-pipe cubic, relative error <= 1e-4, in the numerator
# and the sum) add <= 2e-4 A_e.  fp32 accumulation of S and of the sums is negligible at these sizes.
KC_BOUND = 3 * 2.0 ** -9 + 4e-4


@pytest.mark.parametrize("d,h,m,wq", [(128, 4, 16, 1.0), (128, 4, 64, 1.0), (128, 4, 8, 8.0), (128, 4, 64, 8.0),
                                      (128, 4, 8, 1.0), (128, 4, 5, 1.0), (128, 4, 12, 1.0),
                                      (256, 8, 32, 1.0), (512, 8, 32, 1.0)])
def test_attention_stage_isolated(d, h, m, wq):
    """the attention output Y of one layer against an f64 softmax over the GPU's own
    bf16 U and X~ (read back from the device), elementwise within the arithmetic's rounding bound
    KC_BOUND * A_e (the SURVEY's proposed 4e-3 row-relative bound is below the two bf16 output roundings
    the kernels do: measured 4.4-6.4e-3 row-relative; row-relative <= 1e-2 is kept as a second check).  m h <= 64 takes the
    transposed kernel (its 32-column instantiation for m h <= 32: m = 8 and 5, the latter with partial
    column groups; m = 12 is 48 rows on the 64-column one), 256 the 128-row kernel, d = 256 / 512 the wide kernel; the 9000-key history
    is split into chunks and folded (split-K LSE merge); wq = 8 is the sharp-softmax regime."""
    import torch
    import paper_2511_06077_b200 as stca
    lengths = np.array([9000, 1, 333, 2049])
    cfg = make_cfg(B=len(lengths), m=m, d=d, h=h, M=2)
    wl = workload.make_workload(cfg, seed=21, lengths=lengths, wq_scale=wq)
    c = wl.cfg
    mdl = stca.STCA(workload.full_weights(wl), d=d, h=h, r=c.r, M=c.M, dtype="bf16")
    X, xt = device_inputs(wl)
    NQ = wl.Nt * h
    Ucap = torch.zeros(NQ, d, dtype=torch.int16, device="cuda")
    Ycap = torch.zeros(NQ, d, dtype=torch.int16, device="cuda")
    Z = torch.empty(wl.Nt, c.M, d, device="cuda")
    for layer in (1, 2):
        mdl.project_history(X, wl.hist_off)
        mdl.debug_capture(layer, Ucap, Ycap)
        mdl.forward(xt, wl.tgt_off, Z, None)
        torch.cuda.synchronize()
        U = workload.bits_to_f32(Ucap.cpu().numpy().view(np.uint16)).reshape(NQ, d).astype(np.float64)
        Yg = workload.bits_to_f32(Ycap.cpu().numpy().view(np.uint16)).reshape(NQ, d).astype(np.float64)
        Xc = mdl.read_cache(layer, 0, int(lengths.sum())).astype(np.float64)
        ref, A = _f64_attention(U, Xc, lengths, wl.tgt_off, h)
        assert np.isfinite(Yg).all()
        ratio = np.abs(Yg - ref) / (KC_BOUND * A + 1e-30)
        assert ratio.max() <= 1.0, (layer, ratio.max(), np.unravel_index(ratio.argmax(), ratio.shape))
        e = rowrel(Yg, ref)
        assert e.max() <= 1e-2, (layer, e.max(), int(e.argmax()))
    mdl.close()


@pytest.mark.gpu
@pytest.mark.parametrize("m", [8, 16])
def test_attention_stage_isolated_many_items_per_cta(m):
    """The persistent narrow kernel with several items per CTA (600 requests over <= 148 CTAs), many
    of them one key tile long or a single key: the deferred per-item output (written during the next
    item's first tile) and the O^T double buffer must hand every item its own sums and columns.
    Same bound as test_attention_stage_isolated."""
    import torch
    import paper_2511_06077_b200 as stca
    rng = np.random.default_rng(5)
    lengths = rng.integers(1, 700, 600)
    lengths[::7] = 1
    lengths[3::11] = 128
    cfg = make_cfg(B=len(lengths), m=m, d=128, h=4, M=2)
    wl = workload.make_workload(cfg, seed=23, lengths=lengths)
    c = wl.cfg
    mdl = stca.STCA(workload.full_weights(wl), d=128, h=4, r=c.r, M=c.M, dtype="bf16")
    X, xt = device_inputs(wl)
    NQ = wl.Nt * 4
    Ucap = torch.zeros(NQ, 128, dtype=torch.int16, device="cuda")
    Ycap = torch.zeros(NQ, 128, dtype=torch.int16, device="cuda")
    Z = torch.empty(wl.Nt, c.M, 128, device="cuda")
    mdl.project_history(X, wl.hist_off)
    mdl.debug_capture(2, Ucap, Ycap)
    mdl.forward(xt, wl.tgt_off, Z, None)
    torch.cuda.synchronize()
    U = workload.bits_to_f32(Ucap.cpu().numpy().view(np.uint16)).reshape(NQ, 128).astype(np.float64)
    Yg = workload.bits_to_f32(Ycap.cpu().numpy().view(np.uint16)).reshape(NQ, 128).astype(np.float64)
    Xc = mdl.read_cache(2, 0, int(lengths.sum())).astype(np.float64)
    ref, A = _f64_attention(U, Xc, lengths, wl.tgt_off, 4)
    assert np.isfinite(Yg).all()
    ratio = np.abs(Yg - ref) / (KC_BOUND * A + 1e-30)
    assert ratio.max() <= 1.0, (ratio.max(), np.unravel_index(ratio.argmax(), ratio.shape))
    mdl.close()
