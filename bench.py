"""Bench: targets/sec of the STCA forward under RLB @10k history (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config serve] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...       (one rank per GPU, NCCL)

A step = one pass of the whole hot path over one batch:
stca_project_history (suffix truncation + X~(i) for every layer) then stca_forward
(q(1), M x [U, ragged attention, o(i), fusion], z).  Inputs are resident in HBM when
the timed region starts; X (655 MB at serve) and the X~ cache (2.6 GB) are larger
than the 126 MB L2, so no flush is needed between steps.  Multi-GPU is weak scaling:
every rank runs its own seeded serve-shaped shard, with no collective on the data
path; the time is the max over ranks.  The JSON line carries the roofline of the
dominant kernel (the history projection), the oracle's CPU baseline, the end-to-end
number through the C ABI with host buffers, the launch count and the SM clocks.
"""
from __future__ import annotations

import argparse
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


def algorithmic(wl):
    """Algorithmic work per step: FLOPs / bytes of the method itself."""
    c = wl.cfg
    L = np.minimum(wl.lengths, c.L_infer) if c.L_infer else wl.lengths
    T2 = int(L.sum())
    m = np.diff(wl.tgt_off)
    proj_flops = 6.0 * c.r * c.d * c.d * T2 * c.M                      # 3 GEMMs of d x rd per token per layer
    proj_bytes = 2.0 * c.d * T2 + 2.0 * c.d * T2 * c.M                # read X once, write M layers (bf16)
    attn_flops = float(np.sum(4.0 * m * c.h * c.d * L)) * c.M          # S = U X~^T and Y = P X~
    attn_bytes = float(np.sum(2.0 * c.d * L + 6.0 * m * c.d)) * c.M
    return dict(T2=T2, proj_flops=proj_flops, proj_bytes=proj_bytes, attn_flops=attn_flops, attn_bytes=attn_bytes)


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


def oracle_sample(wl, budget_s=20.0, reps=1):
    """cpu_baseline: the oracle as it stands, threads over requests on the host cores, on a
    bounded deterministic sample (the first k requests, k = cores)."""
    import oracle
    cores = os.cpu_count() or 1
    k = min(cores, len(wl.lengths))
    reqs = list(range(k))
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.forward_workload(wl, requests=reqs, nthreads=cores)
    dt = (time.perf_counter() - t0) / reps
    targets = int(sum(wl.tgt_off[b + 1] - wl.tgt_off[b] for b in reqs))
    return {"value": targets / dt, "unit": UNIT, "cores": min(cores, k), "kind": "oracle",
            "sample": f"first {k} of {len(wl.lengths)} requests ({targets} targets, full history each), "
                      f"{dt:.2f} s per pass"}


def run_reference(args, wl):
    """--impl reference: the f64 oracle timed as the reference arm on host cores."""
    import oracle  # noqa: F401
    cores = os.cpu_count() or 1
    k = min(cores, len(wl.lengths))
    reqs = list(range(k))
    import oracle as orc
    for _ in range(args.warmup):
        orc.forward_workload(wl, requests=reqs, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        orc.forward_workload(wl, requests=reqs, nthreads=cores)
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    targets = int(sum(wl.tgt_off[b + 1] - wl.tgt_off[b] for b in reqs))
    v = targets / dt
    c = wl.cfg
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(wl, args),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": min(cores, k), "kind": "oracle",
                             "sample": f"each step: first {k} of {len(wl.lengths)} requests ({targets} targets)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(wl, args):
    c = wl.cfg
    L = wl.lengths
    return {"workload": c.name, "requests": int(len(L)), "targets_per_request": int(np.diff(wl.tgt_off)[0]),
            "L_avg": float(L.mean()), "L_max": int(L.max()), "L_infer": c.L_infer, "d": c.d, "h": c.h, "r": c.r,
            "M": c.M, "T": wl.T, "N_t": wl.Nt,
            "parallelism": (f"split-history over {args.gpus} GPU(s) (NCCL all-gather of partials per layer)"
                            if c.name == "split1" else f"requests sharded over {args.gpus} GPU(s), weak"),
            "l2": "inputs larger than L2 (X and the X~ cache exceed 126 MB); no flush", "seed": args.seed}


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
    ap.add_argument("--chunk-keys", type=int, default=0, help="split-K chunk cap in keys (0: library default)")
    args = ap.parse_args()
    rank, world, local = env_rank()
    args.gpus = max(args.gpus, world)

    if args.impl == "reference":
        if rank != 0:
            return
        wl = workload.make_workload(args.config, seed=args.seed)
        run_reference(args, wl)
        return

    import torch
    import torch.distributed as dist
    import paper_2511_06077_b200 as stca
    from paper_2511_06077_b200 import _lib

    torch.cuda.set_device(local)
    if world > 1:
        if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
            os.environ["NCCL_DEBUG"] = "WARN"  # stdout carries exactly one JSON line (NCCL prints its version otherwise)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # split1 (BASELINE config 5): ONE L = 10k history split over the ranks (split-history, strong
    # scaling, one all-gather of partials per layer); every other config: each rank its own shard
    split = args.config == "split1"
    wl = workload.make_workload(args.config, seed=args.seed if split else args.seed + 1000 * rank)
    c = wl.cfg
    W = workload.full_weights(workload.make_workload(args.config, seed=args.seed, B=1)) if rank else \
        workload.full_weights(wl)                                            # weights replicated (seed 0 draw)
    model = stca.STCA(W, d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype, with_z=c.with_z,
                      device=local, chunk_keys=1280 if split else args.chunk_keys,
                      split_rank=rank if split else 0, split_world=world if split else 1,
                      exchange=stca.nccl_exchange() if split and world > 1 else None)
    bf16 = c.dtype == "bf16"
    Xh = wl.X_bits.view(np.int16) if bf16 else wl.X
    xth = wl.xt_bits.view(np.int16) if bf16 else wl.xt
    X = torch.from_numpy(Xh).cuda()
    xt = torch.from_numpy(xth).cuda()
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
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.kernel_launches()
    with Clocks(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(st)
        for i in range(K):
            a, b, e = ev[i]
            a.record(st)
            model.project_history(X, wl.hist_off, stream=st)
            b.record(st)
            model.forward(xt, wl.tgt_off, Z, z, stream=st)
            e.record(st)
        t_end.record(st)
        torch.cuda.synchronize()
    launches = (_lib.kernel_launches() - launches0) // max(K, 1)
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end) / K
    proj_ms = [ev[i][0].elapsed_time(ev[i][1]) for i in range(K)]
    fwd_ms = [ev[i][1].elapsed_time(ev[i][2]) for i in range(K)]
    t = torch.tensor([ms, statistics.mean(fwd_ms)], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, fwd_max = float(t[0]), float(t[1])
    total_targets = wl.Nt if split else wl.Nt * world
    value = total_targets / (ms_max * 1e-3)

    # e2e through the C ABI with HOST buffers (pinned), H2D/D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        Xp = torch.from_numpy(Xh).pin_memory()
        xtp = torch.from_numpy(xth).pin_memory()
        Zp = torch.empty(wl.Nt, c.M, c.d).pin_memory()
        zp = torch.empty(wl.Nt, c.d).pin_memory()
        model.project_history(Xp, wl.hist_off, stream=st)
        model.forward(xtp, wl.tgt_off, Zp, zp, stream=st, sync=False)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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
               "d2h_bytes_per_step": int(Zp.numel() * 4 + zp.numel() * 4)}

    if rank == 0:
        pk = peaks()
        alg = algorithmic(wl)
        proj_avg = statistics.mean(proj_ms)
        achieved = alg["proj_flops"] / (proj_avg * 1e-3) / 1e12
        peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tf):
            traffic = json.load(open(tf)).get(c.name, {}).get("projection_dram_bytes_per_launch")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong" if split else "weak",
            "vs_baseline": None,
            "dtype": "bf16" if bf16 else "fp32", "data": "synthetic", "config": config_dict(wl, args),
            "roofline": {"kernel": "history projection (a1, stca_project_history)", "bound": "tensor",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "peak_kind": "measured sustained bf16 (MEASURED_PEAKS.json)",
                         "traffic": traffic, "algorithmic_flops_per_launch": alg["proj_flops"],
                         "ms_per_launch": proj_avg},
            "phases": {"project_ms": proj_avg, "forward_ms": statistics.mean(fwd_ms),
                       "forward_ms_max_over_ranks": fwd_max,
                       "targets_per_s_cached_history": total_targets / (fwd_max * 1e-3),
                       "attention_alg_TFLOP": alg["attn_flops"] / 1e12, "attention_alg_GB": alg["attn_bytes"] / 1e9},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "e2e": e2e,
        }
        if world == 1 and not args.no_oracle:
            line["cpu_baseline"] = oracle_sample(wl)
        print(json.dumps(line), flush=True)
    model.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
