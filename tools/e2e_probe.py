"""e2e diagnostics at the serve config (host buffers through the C ABI).  Diagnostic only."""
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
Xd = Xp.cuda()
xtd = xtp.cuda()
Zd = torch.empty(wl.Nt, c.M, c.d, device="cuda")
zd = torch.empty(wl.Nt, c.d, device="cuda")
st = torch.cuda.current_stream()


def timed(fn, K=6):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(K):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K, (time.perf_counter() - t0) * 1e3 / K


# raw PCIe
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
buf = torch.empty_like(Xd)
zb = torch.empty_like(Zd)


def h2d():
    with torch.cuda.stream(s1):
        buf.copy_(Xp, non_blocking=True)
    st.wait_stream(s1)


def h2d_d2h():
    with torch.cuda.stream(s1):
        buf.copy_(Xp, non_blocking=True)
    with torch.cuda.stream(s2):
        Zp.copy_(zb, non_blocking=True)
    st.wait_stream(s1)
    st.wait_stream(s2)


print("raw H2D 655 MB: %.2f ms" % timed(h2d)[0], flush=True)
print("raw H2D 655 MB + D2H 42 MB concurrently: %.2f ms" % timed(h2d_d2h)[0], flush=True)
m = stca.STCA(W, d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype)
cases = {
    "device in / device out": lambda: (m.project_history(Xd, wl.hist_off, stream=st),
                                       m.forward(xtd, wl.tgt_off, Zd, zd, stream=st)),
    "host X / device xt, out": lambda: (m.project_history(Xp, wl.hist_off, stream=st),
                                        m.forward(xtd, wl.tgt_off, Zd, zd, stream=st)),
    "device X / host xt, out": lambda: (m.project_history(Xd, wl.hist_off, stream=st),
                                        m.forward(xtp, wl.tgt_off, Zp, zp, stream=st, sync=False)),
    "host everything": lambda: (m.project_history(Xp, wl.hist_off, stream=st),
                                m.forward(xtp, wl.tgt_off, Zp, zp, stream=st, sync=False)),
    "host everything + host wait": lambda: (m.project_history(Xp, wl.hist_off, stream=st),
                                            m.forward(xtp, wl.tgt_off, Zp, zp, stream=st, sync=False),
                                            st.synchronize()),
}
for name, fn in cases.items():
    dev, host = timed(fn)
    print(f"{name}: {dev:.2f} ms/step device, {host:.2f} ms/step host = {wl.Nt / dev * 1e3 / 1e6:.3f} M targets/s",
          flush=True)
m.close()
