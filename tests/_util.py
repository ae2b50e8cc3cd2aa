"""Test helpers: run the CUDA path through the C ABI and compare with the oracle."""
import numpy as np

import workload


def rowrel(got, ref):
    """Row-infinity-relative error per (target, layer) row: max_e |g - o| / max_e |o| (R20)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.abs(ref).max(-1)
    den = np.where(den == 0, 1.0, den)
    return np.abs(got - ref).max(-1) / den


def make_cfg(name="t", B=1, m=1, d=128, h=4, r=4, M=4, dtype="bf16", L_infer=0, shared=True, with_z=True):
    return workload.Config(name, B=B, m=m, d=d, h=h, r=r, M=M, dtype=dtype, L_fixed=16, L_infer=L_infer,
                           shared_ffn=shared, with_z=with_z)


def device_inputs(wl, device="cuda"):
    import torch
    if wl.cfg.dtype == "bf16":
        X = torch.from_numpy(wl.X_bits.view(np.int16)).to(device)
        xt = torch.from_numpy(wl.xt_bits.view(np.int16)).to(device)
    else:
        X = torch.from_numpy(np.ascontiguousarray(wl.X)).to(device)
        xt = torch.from_numpy(np.ascontiguousarray(wl.xt)).to(device)
    return X, xt


def run_gpu(wl, *, chunk_keys=0, host=False, model=None, dtype=None):
    """Project + forward through the C ABI; returns (Z, z) as float64 numpy."""
    import torch
    import paper_2511_06077_b200 as stca
    c = wl.cfg
    dtype = dtype or c.dtype
    m = model or stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=dtype,
                           with_z=c.with_z, chunk_keys=chunk_keys)
    if host:
        if dtype == "bf16":
            X, xt = wl.X_bits, wl.xt_bits
        else:
            X, xt = np.ascontiguousarray(wl.X), np.ascontiguousarray(wl.xt)
        Z = np.full((wl.Nt, c.M, c.d), np.nan, dtype=np.float32)
        z = np.full((wl.Nt, c.d), np.nan, dtype=np.float32) if c.with_z else None
        m.project_history(X, wl.hist_off)
        m.forward(xt, wl.tgt_off, Z, z)
        return Z.astype(np.float64), (z.astype(np.float64) if z is not None else None)
    X, xt = device_inputs(wl)
    Z = torch.full((wl.Nt, c.M, c.d), float("nan"), dtype=torch.float32, device="cuda")
    z = torch.full((wl.Nt, c.d), float("nan"), dtype=torch.float32, device="cuda") if c.with_z else None
    m.project_history(X, wl.hist_off)
    m.forward(xt, wl.tgt_off, Z, z)
    torch.cuda.synchronize()
    return Z.cpu().numpy().astype(np.float64), (z.cpu().numpy().astype(np.float64) if z is not None else None)
