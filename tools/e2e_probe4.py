"""Does a pinned H2D copy on a side stream overlap device work on another stream?  Diagnostic only."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workload  # noqa: E402
import paper_2511_06077_b200 as stca  # noqa: E402

wl = workload.make_workload("serve", seed=0, bits_only=True)
c = wl.cfg
Xp = torch.from_numpy(wl.X_bits.view(np.int16)).pin_memory()
Xd = Xp.cuda()
buf = torch.empty_like(Xd)
xtd = torch.from_numpy(wl.xt_bits.view(np.int16)).cuda()
Zd = torch.empty(wl.Nt, c.M, c.d, device="cuda")
zd = torch.empty(wl.Nt, c.d, device="cuda")
m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype)
st = torch.cuda.Stream()
cp = torch.cuda.Stream()
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)


def timed(fn, K=4):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


def copy_only():
    with torch.cuda.stream(cp):
        buf.copy_(Xp, non_blocking=True)


def step_only():
    m.project_history(Xd, wl.hist_off, stream=st)
    m.forward(xtd, wl.tgt_off, Zd, zd, stream=st)


def gemm_only():
    with torch.cuda.stream(st):
        for _ in range(5):
            a @ a


def both(fn):
    def f():
        with torch.cuda.stream(cp):
            buf.copy_(Xp, non_blocking=True)
        fn()
    return f


for name, fn in [("H2D 655 MB", copy_only), ("device step", step_only), ("5 GEMM 8192^3", gemm_only),
                 ("H2D || device step", both(step_only)), ("H2D || 5 GEMM", both(gemm_only))]:
    print(f"{name}: {timed(fn):.2f} ms", flush=True)
m.close()
