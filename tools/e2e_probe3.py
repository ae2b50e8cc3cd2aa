"""Which call blocks the host in the host-input serve loop?  Diagnostic only."""
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
Xp = torch.from_numpy(wl.X_bits.view(np.int16)).pin_memory()
print("pinned:", Xp.is_pinned(), flush=True)
xtd = torch.from_numpy(wl.xt_bits.view(np.int16)).cuda()
Zd = torch.empty(wl.Nt, c.M, c.d, device="cuda")
zd = torch.empty(wl.Nt, c.d, device="cuda")
st = torch.cuda.current_stream()
for alloc in ("torch", "cuda"):
    m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype,
                  allocator=alloc)
    for _ in range(3):
        m.project_history(Xp, wl.hist_off, stream=st)
        m.forward(xtd, wl.tgt_off, Zd, zd, stream=st)
    torch.cuda.synchronize()
    tp, tf = [], []
    for _ in range(6):
        t0 = time.perf_counter()
        m.project_history(Xp, wl.hist_off, stream=st)
        t1 = time.perf_counter()
        m.forward(xtd, wl.tgt_off, Zd, zd, stream=st)
        t2 = time.perf_counter()
        tp.append((t1 - t0) * 1e3)
        tf.append((t2 - t1) * 1e3)
    torch.cuda.synchronize()
    print(alloc, "host ms project:", [round(x, 2) for x in tp], "forward:", [round(x, 2) for x in tf], flush=True)
    # the same with a side stream instead of the legacy default stream
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        for _ in range(2):
            m.project_history(Xp, wl.hist_off, stream=s2)
            m.forward(xtd, wl.tgt_off, Zd, zd, stream=s2)
        s2.synchronize()
        tp = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s2)
        for _ in range(6):
            t0 = time.perf_counter()
            m.project_history(Xp, wl.hist_off, stream=s2)
            m.forward(xtd, wl.tgt_off, Zd, zd, stream=s2)
            tp.append((time.perf_counter() - t0) * 1e3)
        e1.record(s2)
        s2.synchronize()
        print(alloc, "side stream: host ms/step", [round(x, 2) for x in tp], "device ms/step",
              round(e0.elapsed_time(e1) / 6, 2), flush=True)
    m.close()
