"""e2e variants at the serve config (host buffers through the C ABI): allocator torch vs cuda, with and
without a host wait per step.  Diagnostic only."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workload  # noqa: E402
import paper_2511_06077_b200 as stca  # noqa: E402

wl = workload.make_workload("serve", seed=0, bits_only=True)
c = wl.cfg
W = workload.full_weights(wl)
Xp = torch.from_numpy(wl.X_bits.view(np.int16)).pin_memory()
xtp = torch.from_numpy(wl.xt_bits.view(np.int16)).pin_memory()
Zp = torch.empty(wl.Nt, c.M, c.d).pin_memory()
zp = torch.empty(wl.Nt, c.d).pin_memory()
st = torch.cuda.current_stream()
for alloc in ("torch", "cuda"):
    m = stca.STCA(W, d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype, allocator=alloc)
    for hostwait in (False, True):
        for _ in range(2):
            m.project_history(Xp, wl.hist_off, stream=st)
            m.forward(xtp, wl.tgt_off, Zp, zp, stream=st, sync=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 8
        t0 = time.perf_counter()
        e0.record(st)
        for _ in range(K):
            m.project_history(Xp, wl.hist_off, stream=st)
            m.forward(xtp, wl.tgt_off, Zp, zp, stream=st, sync=False)
            if hostwait:
                st.synchronize()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        print(f"allocator={alloc} hostwait={hostwait}: {ms:.2f} ms/step = {wl.Nt / ms * 1e3 / 1e6:.3f} M targets/s "
              f"(host {(time.perf_counter() - t0) * 1e3 / K:.2f} ms/step)", flush=True)
    m.close()
