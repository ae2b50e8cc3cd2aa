"""Two stca_backward calls (the whole-stack backward) at a BASELINE config (default train), for ncu launch
lists of the training step.    python tools/stack_bwd_probe.py [config]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workload  # noqa: E402
import paper_2511_06077_b200 as stca  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "train"
wl = workload.make_workload(cfgname, seed=0, bits_only=True)
c = wl.cfg
m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype)
X = torch.from_numpy(wl.X_bits.view(np.int16)).cuda()
xt = torch.from_numpy(wl.xt_bits.view(np.int16)).cuda()
m.project_history(X, wl.hist_off)
dZ = torch.randn(wl.Nt, c.M, c.d, device="cuda")
dz = torch.randn(wl.Nt, c.d, device="cuda")
grads = {n: torch.empty(tuple(sh), device="cuda") for n, sh in m._shapes.items()}
dX = torch.empty(X.shape[0], c.d, device="cuda")
dxt = torch.empty(wl.Nt, c.d, device="cuda")
Z = torch.empty(wl.Nt, c.M, c.d, device="cuda")
for _ in range(2):
    m.backward(xt, wl.tgt_off, X, dZ, dz, grads=grads, dX=dX, dxt=dxt, out_Z=Z)
torch.cuda.synchronize()
assert torch.isfinite(dX).all()
print("ok", cfgname, X.shape[0], wl.Nt)
m.close()
