"""One project + forward of a BASELINE config subset (for ncu captures of one kernel).
    python tools/attn_case.py <config> <n_requests> [steps]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workload  # noqa: E402
import paper_2511_06077_b200 as stca  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
wl = workload.subset(workload.make_workload(name, seed=0, B=n, bits_only=True), range(n), with_f32=False)
c = wl.cfg
m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype)
X = torch.from_numpy(wl.X_bits.view(np.int16)).cuda()
xt = torch.from_numpy(wl.xt_bits.view(np.int16)).cuda()
Z = torch.empty(wl.Nt, c.M, c.d, device="cuda")
z = torch.empty(wl.Nt, c.d, device="cuda")
for _ in range(steps):
    m.project_history(X, wl.hist_off)
    m.forward(xt, wl.tgt_off, Z, z)
torch.cuda.synchronize()
assert torch.isfinite(Z).all() and torch.isfinite(z).all()
print("ok", name, n, wl.T, wl.Nt)
m.close()
