"""Serve-shaped forward on a subset of requests (profiling aid: ncu -k regex:k_tc_attention)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload, paper_2511_06077_b200 as stca
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
wl = workload.make_workload('serve', seed=0, B=B)
c = wl.cfg
m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer)
X = torch.from_numpy(wl.X_bits.view(np.int16)).cuda()
xt = torch.from_numpy(wl.xt_bits.view(np.int16)).cuda()
Z = torch.empty(wl.Nt, c.M, c.d, device='cuda'); z = torch.empty(wl.Nt, c.d, device='cuda')
m.project_history(X, wl.hist_off)
for _ in range(2):
    m.forward(xt, wl.tgt_off, Z, z)
torch.cuda.synchronize()
print('ok')
