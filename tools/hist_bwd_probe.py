"""One stca_history_backward call at a BASELINE config (default train) for kernel launch lists (ncu)."""
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
m.project_history(X, wl.hist_off)
dXt = torch.randn(X.shape[0], c.d, device="cuda")
dX = torch.zeros(X.shape[0], c.d, device="cuda")
for _ in range(3):
    m.history_backward(1, X, dXt, dX=dX)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
m.history_backward(1, X, dXt, dX=dX)
e1.record()
torch.cuda.synchronize()
print("history_backward ms", e0.elapsed_time(e1), flush=True)
m.close()
