"""GPU parity of the history-path backward (stca_history_backward, NEXT-1 partial; Eq.(1)-(2))
against oracle/history_backward.py on the same bf16 X and weights, chained after the attention backward:
dX~ of every layer comes from stca_attention_backward, dX sums the layers.  The GPU rounds H, dy, dH-derived
da / dg to bf16 for its GEMMs (2^-9 relative each): dX row-inf-relative <= 3e-2; weight gradients (sums over
all rows) relative to their largest entry <= 2e-2."""
import numpy as np
import pytest

import workload
from oracle import attention_backward as ab
from oracle import history_backward as hb
from _util import device_inputs, make_cfg, rowrel

pytestmark = pytest.mark.gpu


def test_history_backward_matches_oracle():
    import torch
    import paper_2511_06077_b200 as stca
    lengths = np.array([300, 1, 2500, 129])
    cfg = make_cfg(B=len(lengths), m=16, M=2)
    wl = workload.make_workload(cfg, seed=61, lengths=lengths, ln_affine=True)
    c = wl.cfg
    mdl = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, dtype="bf16")
    X, xt = device_inputs(wl)
    NQ, T = wl.Nt * c.h, int(lengths.sum())
    Z = torch.empty(wl.Nt, c.M, c.d, device="cuda")
    dX = torch.zeros(T, c.d, device="cuda")
    dXr = np.zeros((T, c.d))
    rng = np.random.default_rng(5)
    for layer in (1, 2):
        U = torch.zeros(NQ, c.d, dtype=torch.int16, device="cuda")
        Y = torch.zeros(NQ, c.d, dtype=torch.int16, device="cuda")
        mdl.project_history(X, wl.hist_off)
        mdl.debug_capture(layer, U, Y)
        mdl.forward(xt, wl.tgt_off, Z, None)
        dY = torch.from_numpy(rng.standard_normal((NQ, c.d)).astype(np.float32)).cuda()
        dXt, _ = mdl.attention_backward(layer, U, dY, wl.tgt_off, dXt=torch.empty(T, c.d, device="cuda"))
        _, g = mdl.history_backward(layer, X, dXt, dX=dX)
        torch.cuda.synchronize()
        w = wl.weights
        ref = hb.backward(wl.X, w[f"L{layer}.hist.Wu"], w[f"L{layer}.hist.Wv"], w[f"L{layer}.hist.Wo"],
                          w[f"L{layer}.hist.ln_g"], w[f"L{layer}.hist.ln_b"], dXt.cpu().double().numpy())
        dXr += ref[0]
        for name, got, want in zip(["Wu", "Wv", "Wo", "ln_g", "ln_b"], [g[k] for k in ("Wu", "Wv", "Wo", "ln_g", "ln_b")],
                                   ref[1:]):
            got = got.cpu().double().numpy().reshape(np.shape(want))
            err = np.abs(got - want).max() / np.abs(want).max()
            assert err <= 2e-2, (layer, name, err)
    e = rowrel(dX.cpu().double().numpy(), dXr)
    assert np.isfinite(e).all() and e.max() <= 3e-2, e.max()
    mdl.close()
