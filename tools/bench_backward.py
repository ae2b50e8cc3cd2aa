"""Measurement of the attention backward (stca_attention_backward, NEXT-1 partial) at a BASELINE config
(default: train, the training shape: 1024 requests x 16 targets, ragged avg 2k / max 4k, d = 128, h = 4).

One launch = one layer's backward over the whole batch.  Algorithmic work per launch:
  FLOPs  sum_b m_b h L'_b (2d [S recomputed] + 2d [dP] + 4d [dX~ = alpha^T dY + dS^T U] + 2d [dU])
  bytes  sum_b (2d L'_b [X~ once] + 4d L'_b [dX~ fp32 out] + m_b h (2d [U] + 4d [dY] + 4d [dU]))
Timed with CUDA events over K launches on the launching stream after warm-up; prints one JSON line.

    python tools/bench_backward.py [--config train] [--steps 10] [--warmup 3]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workload  # noqa: E402
import paper_2511_06077_b200 as stca  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="train")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    wl = workload.make_workload(a.config, seed=0, bits_only=True)
    c = wl.cfg
    m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype)
    X = torch.from_numpy(wl.X_bits.view(np.int16)).cuda()
    xt = torch.from_numpy(wl.xt_bits.view(np.int16)).cuda()
    NQ = wl.Nt * c.h
    U = torch.zeros(NQ, c.d, dtype=torch.int16, device="cuda")
    Y = torch.zeros(NQ, c.d, dtype=torch.int16, device="cuda")
    Z = torch.empty(wl.Nt, c.M, c.d, device="cuda")
    m.project_history(X, wl.hist_off)
    m.debug_capture(1, U, Y)
    m.forward(xt, wl.tgt_off, Z, None)
    L = np.minimum(wl.lengths, c.L_infer) if c.L_infer else wl.lengths
    T2 = int(L.sum())
    dY = torch.randn(NQ, c.d, device="cuda")
    dX = torch.empty(T2, c.d, device="cuda")
    dU = torch.empty(NQ, c.d, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(a.warmup):
        m.attention_backward(1, U, dY, wl.tgt_off, dXt=dX, dU=dU, stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.steps):
        m.attention_backward(1, U, dY, wl.tgt_off, dXt=dX, dU=dU, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    mq = np.diff(wl.tgt_off) * c.h
    flops = float(np.sum(mq * L * 10.0 * c.d))
    byts = float(np.sum(6.0 * c.d * L + mq * 10.0 * c.d))
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
    ridge = pk["bf16_tflops"] * 1e12 / (pk["hbm_gbs"] * 1e9)
    bound = "tensor" if flops / byts >= ridge else "hbm"
    ach = flops / (ms * 1e-3) / 1e12 if bound == "tensor" else byts / (ms * 1e-3) / 1e9
    peak = pk["bf16_tflops"] if bound == "tensor" else pk["hbm_gbs"]
    # the history-path backward of the same layer (stca_history_backward): 18 r d^2 FLOPs per kept row
    # (recompute 6 r d^2 + dWo, dH, dWu, dWv, dX 12 r d^2), tensor-bound
    Xk = X if not c.L_infer else None
    hist = None
    if Xk is not None and int(Xk.shape[0]) == T2:
        dXh = torch.zeros(T2, c.d, device="cuda")
        for _ in range(2):
            m.history_backward(1, Xk, dX, dX=dXh, stream=st)
        torch.cuda.synchronize()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(st)
        for _ in range(3):
            m.history_backward(1, Xk, dX, dX=dXh, stream=st)
        h1.record(st)
        torch.cuda.synchronize()
        hms = h0.elapsed_time(h1) / 3
        hfl = 18.0 * c.r * c.d * c.d * T2
        hist = {"kernel": "history-path backward (stca_history_backward, one layer; cuBLAS GEMMs + kernels)",
                "ms_per_call": hms, "achieved_TFLOPs": hfl / (hms * 1e-3) / 1e12,
                "frac_of_bf16_peak": hfl / (hms * 1e-3) / 1e12 / pk["bf16_tflops"], "algorithmic_flops": hfl}
    # the whole-stack backward (stca_backward: forward with saved U / Y + every layer's backward), one call
    full = None
    if Xk is not None and int(Xk.shape[0]) == T2:
        dZ = torch.randn(wl.Nt, c.M, c.d, device="cuda")
        dz = torch.randn(wl.Nt, c.d, device="cuda")
        grads = {n: torch.empty(tuple(sh), device="cuda") for n, sh in m._shapes.items()}
        dXs = torch.empty(T2, c.d, device="cuda")
        dxts = torch.empty(wl.Nt, c.d, device="cuda")
        Zs = torch.empty(wl.Nt, c.M, c.d, device="cuda")
        for _ in range(2):
            m.backward(xt, wl.tgt_off, Xk, dZ, dz, grads=grads, dX=dXs, dxt=dxts, out_Z=Zs, stream=st)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(st)
        for _ in range(3):
            m.backward(xt, wl.tgt_off, Xk, dZ, dz, grads=grads, dX=dXs, dxt=dxts, out_Z=Zs, stream=st)
        f1.record(st)
        torch.cuda.synchronize()
        fms = f0.elapsed_time(f1) / 3
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(st)
        for _ in range(3):
            m.project_history(X, wl.hist_off, stream=st)
        p1.record(st)
        torch.cuda.synchronize()
        pms = p0.elapsed_time(p1) / 3
        full = {"call": "stca_backward (forward keeping U / Y, then the backward of all layers: target side, "
                        "attention, history path; every weight role, dX, dx_t)",
                "ms_per_call": fms, "project_ms": pms,
                "train_step_ms": pms + fms, "train_targets_per_s": wl.Nt / ((pms + fms) * 1e-3),
                "timing": "CUDA events on the launching stream, 3 calls after 2 warm-up calls"}
    print(json.dumps({"kernel": "attention backward (stca_attention_backward, one layer)", "config": a.config,
                      "ms_per_launch": ms, "targets_per_s": wl.Nt / (ms * 1e-3),
                      "roofline": {"bound": bound, "achieved": ach, "peak": peak,
                                   "unit": "TFLOP/s" if bound == "tensor" else "GB/s", "frac": ach / peak,
                                   "algorithmic_flops": flops, "algorithmic_bytes": byts,
                                   "note": "the kernel reads X~ twice (pass 1: softmax statistics; pass 2: "
                                           "gradients): algorithmic bytes count it once"},
                      "T": T2, "N_t": wl.Nt, "history_backward": hist, "stack_backward": full}), flush=True)
    m.close()


if __name__ == "__main__":
    main()
