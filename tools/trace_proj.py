import os, sys, numpy as np, torch
sys.path.insert(0, '.')
import workload, paper_2511_06077_b200 as stca
wl = workload.make_workload('serve', seed=0, B=64)
c = wl.cfg
m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer)
X = torch.from_numpy(wl.X_bits.view(np.int16)).cuda()
for i in range(3):
    m.project_history(X, wl.hist_off)
torch.cuda.synchronize()
os.environ['STCA_TRACE'] = 'gpurun_out/trace_proj.bin'
m.project_history(X, wl.hist_off)
torch.cuda.synchronize()
print('ok')
