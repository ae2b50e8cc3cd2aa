"""Bench: targets/sec of the STCA forward under RLB @10k history (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config serve] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...       (one rank per GPU, NCCL)

A step = one pass of the whole hot path over one batch:
stca_project_history (suffix truncation + X~(i) for every layer) then stca_forward
(q(1), M x [U, ragged attention, o(i), fusion], z).  Inputs are resident in HBM when
the timed region starts; X (655 MB at serve) and the X~ cache (2.6 GB) are larger
than the 126 MB L2, so no flush is needed between steps.

Multi-GPU is STRONG scaling: every rank draws the same
global request set (seed), partitions it with the library's LPT planner
(stca_plan_shards over the cost c_b = L'_b 6rd^2M + m_b L'_b 4hdM + m_b c_tgt) and
runs its own requests; there is no collective on the data path.  value = the global
N_t / the max over ranks of the device time of a step.  `--config split1` runs the
split-history path (one 10k history over all ranks; per layer the partials are read in place from the
owners' buffers over peer memory, or all-gathered by NCCL with --split-exchange nccl).

The JSON line carries the roofline of the projection AND of the attention kernel
(per-phase CUDA events recorded by the library on the launching stream, in a
separate profiled pass after the timed one), the oracle's CPU baseline, the
end-to-end number through the C ABI with host buffers, the launch count and the
SM clocks sampled during the timed region.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workload  # noqa: E402  (seeded inputs; no method arithmetic)

METRIC = "targets/sec STCA fwd @10k history"
UNIT = "targets/s"


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "_fallback": True}


# ---------------------------------------------------------------------------
# request sharding (PAR1): LPT over the per-request cost of SURVEY §8(e)
# ---------------------------------------------------------------------------
def request_cost(wl) -> np.ndarray:
    """c_b = L'_b (6 r d^2 M) + m_b L'_b (4 h d M) + m_b c_tgt, c_tgt = sum_i (6r + 8 + 2(i+1)) d^2
    (FLOPs: history projection, attention, target side; exact int64)."""
    c = wl.cfg
    L = np.minimum(wl.lengths, c.L_infer) if c.L_infer else wl.lengths.copy()
    m = np.diff(wl.tgt_off)
    c_tgt = sum((6 * c.r + 8 + 2 * (i + 1)) * c.d * c.d for i in range(1, c.M + 1))
    return (L * (6 * c.r * c.d * c.d * c.M) + m * L * (4 * c.h * c.d * c.M) + m * c_tgt).astype(np.int64)


def shard_requests(wl, world: int, rank: int) -> np.ndarray:
    """The requests rank `rank` of `world` owns, in generation order (stca_plan_shards, identical on
    every rank: integer costs, ties to the lowest index)."""
    if world <= 1:
        return np.arange(len(wl.lengths), dtype=np.int64)
    from paper_2511_06077_b200 import _lib
    part = _lib.plan_shards(request_cost(wl), world)
    return np.nonzero(part == rank)[0].astype(np.int64)


def algorithmic(wl):
    """Algorithmic work per step: FLOPs / bytes of the method itself."""
    c = wl.cfg
    L = np.minimum(wl.lengths, c.L_infer) if c.L_infer else wl.lengths
    T2 = int(L.sum())
    m = np.diff(wl.tgt_off)
    proj_flops = 6.0 * c.r * c.d * c.d * T2 * c.M                      # 3 GEMMs of d x rd per token per layer
    proj_bytes = 2.0 * c.d * T2 + 2.0 * c.d * T2 * c.M                # read X once, write M layers (bf16)
    # attention, PER LAYER (one a4 launch): S = U X~^T and Y = P X~; bytes = X~ once + q in / o out (fused minimum)
    attn_flops = float(np.sum(4.0 * m * c.h * c.d * L))
    attn_bytes = float(np.sum(2.0 * c.d * L + 6.0 * m * c.d))
    return dict(T2=T2, proj_flops=proj_flops, proj_bytes=proj_bytes, attn_flops_layer=attn_flops,
                attn_bytes_layer=attn_bytes)


class Clocks:
    """SM clocks and clock-event reasons sampled (NVML, every 10 ms, in a thread) DURING the
    timed region -- the B200_PROFILING.md clocks line."""

    def __init__(self, dev):
        self.dev, self.samples, self._stop, self._t = dev, [], None, None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._stop = threading.Event()
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap,
                    "hw_power_brake_slowdown": pynvml.nvmlClocksEventReasonHwPowerBrakeSlowdown}

            def run():
                while not self._stop.is_set():
                    try:
                        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((mhz, [k for k, b in bits.items() if rs & b]))
                    except Exception:
                        pass
                    self._stop.wait(0.01)
            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *a):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return None
        return {"sm_mhz": statistics.median(s[0] for s in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted({r for s in self.samples for r in s[1]}), "samples": len(self.samples),
                "source": "NVML, 10 ms, during the timed region"}


# The oracle's work for one request in f64 multiply-adds (the standard form it computes, Eq.(2)-(9)):
# per layer, the history FFN 3 r d^2 and K / V 2 d^2 per history row, scores and values 2 d per
# (target, row).  ORACLE_MACS_PER_S (one host core, measured: the serve sample, 16 requests of
# 9.8e9 MACs each on 16 threads in 4.76 s) is used only to SIZE the sample, never in a value.
ORACLE_MACS_PER_S = 2.0e9


def _oracle_cost(wl, b):
    c = wl.cfg
    L = int(wl.lengths[b])
    if c.L_infer:
        L = min(L, c.L_infer)
    m = int(wl.tgt_off[b + 1] - wl.tgt_off[b])
    return c.M * (L * (3 * c.r + 2) * c.d ** 2 + m * L * 2 * c.d)


def oracle_subset(wl, budget_s=20.0):
    """The oracle's bounded sample: the first k = cores requests (threads over requests); when one
    pass over them would exceed ``budget_s`` (the capacity config: a 10k history at d = 512 is ~150 s
    of f64 work on one core), the first k requests whose history is at most L_cap, L_cap halved from
    the longest history until the pass fits.  Returns (subset, k, L_cap or None, scale): ``scale``
    converts the sample's targets/s to the whole workload's by the exact per-request cost model
    above (the oracle's cost per target of the sample over that of the workload; 1 without a cap)."""
    cores = os.cpu_count() or 1
    B = len(wl.lengths)
    cost = [_oracle_cost(wl, b) for b in range(B)]

    def pass_s(reqs):
        if not reqs:
            return 0.0
        return max(max(cost[b] for b in reqs), sum(cost[b] for b in reqs) / cores) / ORACLE_MACS_PER_S

    reqs, cap = list(range(min(cores, B))), None
    L_cap = int(wl.lengths.max())
    while pass_s(reqs) > budget_s and L_cap > 64:
        L_cap //= 2
        cap = L_cap
        reqs = [b for b in range(B) if wl.lengths[b] <= L_cap][:cores]
    scale = 1.0
    if cap is not None:
        per_t = lambda rs: sum(cost[b] for b in rs) / max(1, sum(int(wl.tgt_off[b + 1] - wl.tgt_off[b]) for b in rs))
        scale = per_t(reqs) / per_t(range(B))
    return workload.subset(wl, reqs), len(reqs), cap, scale


def _sample_text(wl, k, cap, scale):
    if cap is None:
        return f"first {k} of {len(wl.lengths)} requests (full history each)"
    return (f"first {k} of {len(wl.lengths)} requests with a history of at most {cap} rows (one full pass over "
            f"the first {k} requests would exceed the time bound); targets/s scaled by {scale:.4f} = the oracle's "
            f"cost per target on the sample / on the whole workload (exact f64 multiply-add count)")


def oracle_sample(wl, budget_s=20.0):
    """cpu_baseline: the oracle as it stands, threads over requests on the host cores, on a
    bounded deterministic sample (oracle_subset)."""
    import oracle
    cores = os.cpu_count() or 1
    sub, k, cap, scale = oracle_subset(wl, budget_s)
    t0 = time.perf_counter()
    oracle.forward_workload(sub, nthreads=cores)
    dt = time.perf_counter() - t0
    targets = sub.Nt
    out = {"value": targets / dt * scale, "unit": UNIT, "cores": min(cores, k), "kind": "oracle",
           "sample": f"{_sample_text(wl, k, cap, scale)}: {targets} targets, {dt:.2f} s per pass"}
    if cap is not None:
        out["sample_value"] = targets / dt
    return out


def run_reference(args, wl):
    """--impl reference: the f64 oracle timed as the reference arm on host cores."""
    import oracle as orc
    cores = os.cpu_count() or 1
    sub, k, cap, scale = oracle_subset(wl, budget_s=20.0)
    for _ in range(args.warmup):
        orc.forward_workload(sub, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        orc.forward_workload(sub, nthreads=cores)
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    targets = sub.Nt
    v = targets / dt * scale
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(wl, args),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": min(cores, k), "kind": "oracle",
                             "sample": f"each step: {_sample_text(wl, k, cap, scale)} ({targets} targets)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def e2e_from_ids(model, wl, xth, K, st, world, total_targets):
    """Pinned host ids -> H2D (non-blocking, on the stream) -> stca_encode_history -> project -> forward ->
    D2H of Z and z, K pipelined steps, CUDA events on the stream, max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_2511_06077_b200 as stca
    c = wl.cfg
    g = torch.Generator(device="cuda").manual_seed(11)
    n_video, n_action, n_pos, n_td = 1 << 20, 16, max(c.L_infer or 0, int(wl.lengths.max())), 32
    tab = lambda n: (torch.randn(n, c.d, device="cuda", generator=g) * 0.05).to(torch.bfloat16).view(torch.int16)
    video, action, position, tdelta = tab(n_video + 1), tab(n_action + 1), tab(n_pos), tab(n_td)
    rng = np.random.default_rng(12)
    T, B = wl.T, len(wl.lengths)
    vid = torch.from_numpy(rng.integers(0, n_video + n_video // 100, T)).pin_memory()  # ~1 % out of vocabulary
    act = torch.from_numpy(rng.integers(0, n_action, T)).pin_memory()
    req = torch.from_numpy(np.full(B, 1_700_000_000, dtype=np.int64)).pin_memory()
    ts = torch.from_numpy(1_700_000_000 - rng.integers(0, 1 << 24, T)).pin_memory()
    hoff = torch.from_numpy(np.asarray(wl.hist_off, dtype=np.int64)).pin_memory()
    xtp = torch.from_numpy(np.ascontiguousarray(xth)).pin_memory()
    Zp = torch.empty(wl.Nt, c.M, c.d).pin_memory()
    zp = torch.empty(wl.Nt, c.d).pin_memory()
    # ids travel on a copy stream into two device buffer sets, so step k + 1's upload overlaps step k
    dvs = [[torch.empty_like(a, device="cuda") for a in (vid, act, ts, hoff, req)] for _ in range(2)]
    X = torch.empty(T, c.d, dtype=torch.int16, device="cuda")
    cs = torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    k_ = [0]

    def step():
        b_ = k_[0] & 1
        k_[0] += 1
        dv = dvs[b_]
        cs.wait_event(ev_free[b_])  # encode of two steps ago has read this buffer set
        with torch.cuda.stream(cs):
            for a, b in zip((vid, act, ts, hoff, req), dv):
                b.copy_(a, non_blocking=True)
            ev_in[b_].record(cs)
        st.wait_event(ev_in[b_])
        stca.encode_history(video, action, position, dv[0], dv[1], dv[3], tdelta=tdelta, timestamp=dv[2],
                            req_time=dv[4], X=X, stream=st)
        ev_free[b_].record(st)
        model.project_history(X, wl.hist_off, stream=st)
        model.forward(xtp, wl.tgt_off, Zp, zp, stream=st, sync=False)

    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    device_align(world)
    e0.record(st)
    for _ in range(K):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / K], device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    h2d = sum(a.numel() * a.element_size() for a in (vid, act, ts, hoff, req)) + xtp.numel() * xtp.element_size()
    return {"value": total_targets / (float(te[0]) * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(Zp.numel() * 4 + zp.numel() * 4),
            "input": "raw history ids (video, action, timestamp: 24 B per row) + x_t; X encoded on the device "
                     "(stca_encode_history: video 2^20 + OOV, action 16, position, log2-time-delta tables, bf16, "
                     "resident) then projected",
            "per": "rank 0's shard bytes; time = max over ranks" if world > 1 else "the whole step"}


def device_align(world):
    """Aligns the ranks' STREAMS (not only their hosts) right before a timed region: a one-element
    all-reduce on the current stream completes on every device at about the same time, so host launch
    skew after the barrier does not enter the device-timed region (it would whenever the ranks' kernels
    wait for each other, as split-history's do)."""
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.all_reduce(torch.ones(1, device="cuda"))


def config_dict(wl, args):
    c = wl.cfg
    L = wl.lengths
    return {"workload": c.name, "requests": int(len(L)), "targets_per_request": int(np.diff(wl.tgt_off)[0]),
            "L_avg": float(L.mean()), "L_max": int(L.max()), "L_infer": c.L_infer, "d": c.d, "h": c.h, "r": c.r,
            "M": c.M, "T": wl.T, "N_t": wl.Nt,
            "parallelism": (f"split-history over {args.gpus} GPU(s) ("
                            + ("partials read in place over peer memory, device-side epoch flags"
                               if args.split_exchange == "peer" else "NCCL all-gather of partials per layer") + ")"
                            if c.name == "split1" else
                            f"one global request set, LPT-sharded over {args.gpus} GPU(s) (stca_plan_shards), "
                            "no collective on the data path"),
            "l2": "inputs larger than L2 (X and the X~ cache exceed 126 MB); no flush", "seed": args.seed,
            **({"attention_form": args.form} if args.form != "reordered" else {})}


def lib_sha256():
    from paper_2511_06077_b200 import _lib
    h = hashlib.sha256()
    with open(_lib.LIB_PATH, "rb") as f:
        h.update(f.read())
    return h.hexdigest()


def src_sha256():
    from paper_2511_06077_b200 import build as _b
    return _b.source_digest()


def ncu_for(config, kernel):
    """The committed ncu launch-list summary (profiles/ncu_r2.json, tools/ncu_summary.py) of `kernel` at
    `config` -- only if that capture ran a build of THESE sources (source digest, or the same binary),
    else None."""
    tf = os.path.join(ROOT, "profiles", "ncu_r2.json")
    try:
        t = json.load(open(tf)).get(config, {})
        if t.get("src_sha256") == src_sha256() or t.get("lib_sha256") == lib_sha256():
            return dict(t.get(kernel, {}), source=t.get("source"))
    except Exception:
        pass
    return None


def roofline_entry(name, kernel, flops, bytes_, ms, pk, peak_kind, config):
    """Bound by intensity against the ridge of the peaks in use; achieved = algorithmic work per launch
    / event-timed launch duration."""
    tf_peak = pk["bf16_tflops"] if peak_kind == "burst" else pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    bw_peak = pk["hbm_gbs"]
    ridge = tf_peak * 1e12 / (bw_peak * 1e9)
    intensity = flops / bytes_ if bytes_ else float("inf")
    tensor = intensity >= ridge

    def rate(t_ms):
        return flops / (t_ms * 1e-3) / 1e12 if tensor else bytes_ / (t_ms * 1e-3) / 1e9
    achieved = rate(ms)
    peak, unit, bound = (tf_peak, "TFLOP/s", "tensor") if tensor else (bw_peak, "GB/s", "hbm")
    nc = ncu_for(config, kernel)
    traffic = ncu_ms = None
    if nc and nc.get("ms_per_launch"):
        traffic = nc["dram_bytes_read_per_launch"] + nc["dram_bytes_write_per_launch"]
        ncu_ms = nc["ms_per_launch"]
    return {"kernel": name, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak, "traffic": traffic,
            "ncu": None if ncu_ms is None else {"ms_per_launch": ncu_ms, "achieved": rate(ncu_ms),
                                                "frac": rate(ncu_ms) / peak, "source": nc.get("source"),
                                                "note": "cold-cache, serialised launch list of this build"},
            "peak_kind": f"measured {peak_kind} (MEASURED_PEAKS.json)" + (" (fallback)" if pk.get("_fallback") else ""),
            "algorithmic_flops_per_launch": flops, "algorithmic_bytes_per_launch": bytes_,
            "intensity_flop_per_byte": intensity, "ridge": ridge, "ms_per_launch": ms}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="serve")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="skip the per-phase profiled pass")
    ap.add_argument("--chunk-keys", type=int, default=0, help="split-K chunk cap in keys (0: library default)")
    ap.add_argument("--form", choices=("reordered", "standard"), default="reordered",
                    help="attention form: the paper's reordered Eq.(13) (default) or the standard Eq.(12) with K/V "
                         "per head materialised (NEXT-3 variant, A/B)")
    ap.add_argument("--split-exchange", choices=("peer", "nccl"), default="peer",
                    help="split1 on > 1 GPU: partials read in place over peer memory (stca_split_peer_*, default) "
                         "or all-gathered by NCCL through the exchange callback")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local = env_rank()
    args.gpus = max(args.gpus, world)

    if args.impl == "reference":
        if rank != 0:
            return
        wl = workload.make_workload(args.config, seed=args.seed, bits_only=True)
        run_reference(args, wl)
        return

    import torch
    import torch.distributed as dist
    import paper_2511_06077_b200 as stca
    from paper_2511_06077_b200 import _lib

    torch.cuda.set_device(local)
    if world > 1:
        if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
            os.environ["NCCL_DEBUG"] = "WARN"
        # stdout carries exactly one JSON line: NCCL's version banner goes to stderr (fd 1 -> fd 2 while
        # the communicator is created)
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    # split1 (BASELINE config 5): ONE L = 10k history split over the ranks (split-history, one all-gather
    # of partials per layer); every other config: the same global request set on every rank, LPT-sharded
    split = args.config == "split1"
    gwl = workload.make_workload(args.config, seed=args.seed, bits_only=True)  # the global request set
    c = gwl.cfg
    mine = np.arange(len(gwl.lengths)) if split else shard_requests(gwl, world, rank)
    wl = gwl if (split or world == 1) else workload.subset(gwl, mine, with_f32=False)  # this rank's requests
    W = workload.full_weights(gwl)                                       # weights replicated
    model = stca.STCA(W, d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype, with_z=c.with_z,
                      device=local, chunk_keys=1280 if split else args.chunk_keys,
                      split_rank=rank if split else 0, split_world=world if split else 1,
                      exchange=stca.nccl_exchange() if split and world > 1 and args.split_exchange == "nccl" else None)
    if args.form != "reordered":
        model.set_attention_form(args.form)
    if split and world > 1 and args.split_exchange == "peer":  # partials read in place over NVLink
        model.split_peer_setup(64 << 20)
    bf16 = c.dtype == "bf16"
    Xh = wl.X_bits.view(np.int16) if bf16 else wl.X
    xth = wl.xt_bits.view(np.int16) if bf16 else wl.xt
    X = torch.from_numpy(np.ascontiguousarray(Xh)).cuda()
    xt = torch.from_numpy(np.ascontiguousarray(xth)).cuda()
    Z = torch.empty(wl.Nt, c.M, c.d, device="cuda")
    z = torch.empty(wl.Nt, c.d, device="cuda")
    st = torch.cuda.current_stream()

    def step():
        model.project_history(X, wl.hist_off, stream=st)
        model.forward(xt, wl.tgt_off, Z, z, stream=st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    K = args.steps
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.kernel_launches()
    with Clocks(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        device_align(world)
        t_start.record(st)
        for _ in range(K):
            step()
        t_end.record(st)
        torch.cuda.synchronize()
    launches = (_lib.kernel_launches() - launches0) // max(K, 1)
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end) / K

    # profiled pass (separate from the timed one): per-phase CUDA events on the launching stream
    prof = None
    if not args.no_profile:
        model.profile(True)
        Kp = max(1, min(K, 10))
        for _ in range(Kp):
            step()
        prof = {k: (v[0] / Kp, v[1] // Kp) for k, v in model.profile_read().items()}  # per step: (ms, regions)
        model.profile(False)

    t = torch.tensor([ms, prof["forward"][0] if prof else 0.0, prof["project"][0] if prof else 0.0,
                      len(mine), wl.Nt, wl.T], dtype=torch.float64, device="cuda")
    if world > 1:
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
    else:
        allt = [t]
    per_rank = [[float(x) for x in a.cpu()] for a in allt]
    ms_max = max(r[0] for r in per_rank)
    total_targets = gwl.Nt
    value = total_targets / (ms_max * 1e-3)

    # e2e through the C ABI with HOST buffers (pinned), H2D/D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        Xp = torch.from_numpy(np.ascontiguousarray(Xh)).pin_memory()
        xtp = torch.from_numpy(np.ascontiguousarray(xth)).pin_memory()
        Zp = torch.empty(wl.Nt, c.M, c.d).pin_memory()
        zp = torch.empty(wl.Nt, c.d).pin_memory()
        model.project_history(Xp, wl.hist_off, stream=st)
        model.forward(xtp, wl.tgt_off, Zp, zp, stream=st, sync=False)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        device_align(world)
        e0.record(st)
        for _ in range(K):  # pipelined serving loop: nothing waits on the host inside it
            model.project_history(Xp, wl.hist_off, stream=st)
            model.forward(xtp, wl.tgt_off, Zp, zp, stream=st, sync=False)
        e1.record(st)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / K], device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": total_targets / (float(te[0]) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(Xp.numel() * Xp.element_size() + xtp.numel() * xtp.element_size()),
               "d2h_bytes_per_step": int(Zp.numel() * 4 + zp.numel() * 4),
               "per": "rank 0's shard bytes; time = max over ranks" if world > 1 else "the whole step"}

    # e2e from RAW IDS (NEXT-4): per step the host sends each history row's (video id, action id,
    # timestamp) -- 24 bytes instead of the 2d-byte embedding row -- and the library's encoding prologue
    # (stca_encode_history) builds X on the device from resident tables.  Same pipelined
    # loop and timing as e2e; a secondary field (the values of X differ from the main workload's).
    e2e_ids = None
    if not args.no_e2e and bf16 and not split:
        e2e_ids = e2e_from_ids(model, wl, xth, K, st, world, total_targets)

    if rank == 0:
        pk = peaks()
        clocks = clk.summary()
        reasons = (clocks or {}).get("reasons", [])
        # burst peak for a short timed region at full clocks; sustained if the power cap engaged
        timed_s = ms * K * 1e-3
        peak_kind = "sustained" if ("sw_power_cap" in reasons or timed_s > 1.0) else "burst"
        alg = algorithmic(wl)  # rank 0's shard
        kernels = []
        if prof:  # CUDA-event regions on the launching stream around each projection / attention launch
            if prof["project"][1]:
                kernels.append(roofline_entry("history projection (a1, k_tc_project)", "project", alg["proj_flops"],
                                              alg["proj_bytes"], prof["project"][0] / prof["project"][1], pk,
                                              peak_kind, c.name))
            if prof["attention"][1]:
                # the committed ncu summaries are captures of the reordered form: no attention entry for another
                kernels.append(roofline_entry("ragged single-query attention (a4, one layer)", "attention",
                                              alg["attn_flops_layer"], alg["attn_bytes_layer"],
                                              prof["attention"][0] / prof["attention"][1], pk, peak_kind,
                                              c.name if args.form == "reordered" else f"{c.name}/{args.form}"))
            for k in kernels:
                k["timing"] = ("CUDA events on the launching stream around the launch, K steps after the timed "
                               "region (an upper bound of the kernel time: the events also hold its launch and "
                               "take away the programmatic-dependent-launch overlap)")
        step_ms_prof = (prof["project"][0] + prof["forward"][0]) if prof else None
        dom = None
        if kernels:  # the dominant kernel by time share of the step
            dom = max(kernels, key=lambda k: k["ms_per_launch"] * (1 if "projection" in k["kernel"] else c.M))
        roofline = dict(dom) if dom else None
        if roofline is not None:
            roofline["kernels"] = kernels
            roofline["attention"] = next((k for k in kernels if "attention" in k["kernel"]), None)
        phases = None
        if prof:
            phases = {"project_ms": prof["project"][0], "forward_ms": prof["forward"][0],
                      "attention_ms_per_layer": prof["attention"][0] / max(prof["attention"][1], 1),
                      "merge_ms_per_layer": prof["merge"][0] / max(prof["merge"][1], 1) if prof["merge"][1] else 0.0,
                      "targets_per_s_cached_history": wl.Nt / (prof["forward"][0] * 1e-3),
                      "source": "stca_profile events on the launching stream (separate pass; an upper bound of "
                                "the unprofiled step: events break programmatic-dependent-launch overlap)",
                      "step_ms_profiled": step_ms_prof}
        loads = [r[0] for r in per_rank]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": "bf16" if bf16 else "fp32", "data": "synthetic", "config": config_dict(gwl, args),
            "roofline": roofline,
            "phases": phases,
            "ranks": {"ms_per_step": loads, "requests": [int(r[3]) for r in per_rank],
                      "targets": [int(r[4]) for r in per_rank], "history_rows": [int(r[5]) for r in per_rank],
                      "imbalance_max_over_mean": max(loads) / (sum(loads) / len(loads))},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "e2e": e2e,
            "e2e_ids": e2e_ids,
            "lib_sha256": lib_sha256()[:16],
            "src_sha256": src_sha256()[:16],
        }
        if world == 1 and not args.no_oracle:
            line["cpu_baseline"] = oracle_sample(gwl)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()  # every rank is done with the split-history peer buffers before any handle goes
    model.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
