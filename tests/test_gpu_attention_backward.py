"""GPU parity of the attention backward with request-level gradient aggregation (stca_attention_backward,
NEXT-1 partial) against oracle/attention_backward.py, on the GPU's own bf16 U and X~
(read back from the device) and the same fp32 dY.  Tolerance: the kernel rounds P, dS and dY to bf16 for
its MMAs (relative 2^-9 each) -- row-inf-relative <= 2e-2, the bf16 bound of DESIGN.md R20."""
import numpy as np
import pytest

import workload
from oracle import attention_backward as ab
from _util import device_inputs, make_cfg, rowrel

pytestmark = pytest.mark.gpu


def _run(lengths, m, seed, layer=1, L_infer=0, wq=1.0):
    import torch
    import paper_2511_06077_b200 as stca
    cfg = make_cfg(B=len(lengths), m=m, M=2, L_infer=L_infer)
    wl = workload.make_workload(cfg, seed=seed, lengths=np.asarray(lengths), wq_scale=wq)
    c = wl.cfg
    mdl = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype="bf16")
    X, xt = device_inputs(wl)
    NQ = wl.Nt * c.h
    Ucap = torch.zeros(NQ, c.d, dtype=torch.int16, device="cuda")
    Ycap = torch.zeros(NQ, c.d, dtype=torch.int16, device="cuda")
    Z = torch.empty(wl.Nt, c.M, c.d, device="cuda")
    mdl.project_history(X, wl.hist_off)
    mdl.debug_capture(layer, Ucap, Ycap)
    mdl.forward(xt, wl.tgt_off, Z, None)
    kept = np.minimum(np.asarray(lengths), L_infer) if L_infer else np.asarray(lengths)
    T2 = int(kept.sum())
    dY = torch.from_numpy(np.random.default_rng(seed + 1).standard_normal((NQ, c.d)).astype(np.float32)).cuda()
    dXt = torch.full((T2, c.d), float("nan"), device="cuda")
    dU = torch.full((NQ, c.d), float("nan"), device="cuda")
    mdl.attention_backward(layer, Ucap, dY, wl.tgt_off, dXt=dXt, dU=dU)
    torch.cuda.synchronize()
    U = workload.bits_to_f32(Ucap.cpu().numpy().view(np.uint16)).reshape(NQ, c.d).astype(np.float64)
    Xc = mdl.read_cache(layer, 0, T2).astype(np.float64)
    q_off = np.asarray(wl.tgt_off) * c.h
    dXr, dUr = ab.backward(U, Xc, dY.cpu().double().numpy(), kept, q_off)
    mdl.close()
    return dXt.cpu().double().numpy(), dU.cpu().double().numpy(), dXr, dUr


@pytest.mark.parametrize("m", [16, 8, 33])
def test_attention_backward_matches_oracle(m):
    """m h = 64 (one item per request), 32 (a partial block), 132 (three blocks, fp32 reductions); ragged
    histories incl. one row, a partial last key tile and a 9000-key history."""
    dX, dU, dXr, dUr = _run([300, 1, 9000, 129], m, seed=40 + m)
    assert np.isfinite(dX).all() and np.isfinite(dU).all()
    ex, eu = rowrel(dX, dXr), rowrel(dU, dUr)
    assert ex.max() <= 2e-2, (ex.max(), int(ex.argmax()))
    assert eu.max() <= 2e-2, (eu.max(), int(eu.argmax()))


def test_attention_backward_sharp_and_suffix():
    """Sharp softmax (W_Q x 8) and the serving suffix (L_infer): the cache rows are the kept suffix."""
    dX, dU, dXr, dUr = _run([5000, 70, 2000], 16, seed=7, L_infer=1500, wq=8.0)
    assert rowrel(dX, dXr).max() <= 2e-2 and rowrel(dU, dUr).max() <= 2e-2


def test_single_row_history_aggregates_all_targets():
    """L_b = 1: alpha = 1, so the row's gradient is the sum of every target-head row's dY (the request-level
    aggregation, exactly up to bf16 rounding of dY) and dU = 0."""
    dX, dU, dXr, dUr = _run([1, 1], 16, seed=3)
    assert rowrel(dX, dXr).max() <= 1e-2
    assert np.abs(dU).max() <= 1e-6
