"""Run the fused projection on a small serve-shaped problem (debug aid: compute-sanitizer / hangs)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import workload, paper_2511_06077_b200 as stca
B = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = workload.make_workload('serve', seed=0, B=B, lengths=np.full(B, int(sys.argv[2]) if len(sys.argv) > 2 else 1000))
c = wl.cfg
m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer)
X = torch.from_numpy(wl.X_bits.view(np.int16)).cuda()
m.project_history(X, wl.hist_off)
torch.cuda.synchronize()
print('ok', B)
