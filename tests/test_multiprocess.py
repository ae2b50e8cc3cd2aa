"""World-size-2 tests of the multi-GPU host logic on CPU (gloo): request sharding (PAR1, no
collective on the data path) and the split-history exchange protocol (PAR3).  The device
side runs under `pytest -m gpu` (tests/test_gpu_split.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workload


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_06077_b200 as stca
        out = {}
        # PAR1: every rank computes the same LPT plan from the global request list, independently
        wl = workload.make_workload("multi", seed=3, B=512)
        c = wl.cfg
        L = np.minimum(wl.lengths, c.L_infer)
        m = np.diff(wl.tgt_off)
        cost = L * (6 * c.r * c.d * c.d * c.M) + m * L * (4 * c.h * c.d * c.M)
        plan = torch.from_numpy(stca.plan_shards(cost, world).astype(np.int64))
        plans = [torch.zeros_like(plan) for _ in range(world)]
        dist.all_gather(plans, plan)
        out["plans_equal"] = all(torch.equal(p, plans[0]) for p in plans)
        mine = np.nonzero(plan.numpy() == rank)[0]
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([len(mine)]))
        out["covered"] = int(sum(int(s) for s in sizes)) == len(cost)
        loads = [int(cost[plan.numpy() == r].sum()) for r in range(world)]
        out["balance"] = max(loads) / (sum(loads) / world)
        # PAR3: rank-major all-gather of per-rank partial buffers; chunk c is taken from rank floor(cG/C)
        Lh, cap = 10000, 1280
        n, cl = stca.plan_chunks(Lh, cap)
        o0, ol = stca.plan_split(Lh, cap, world, rank)
        part = torch.full((n,), -1.0)
        for ch in range(o0 // cl, (o0 + ol + cl - 1) // cl):
            part[ch] = float(ch)  # this rank's partial for chunk ch
        gathered = torch.empty(world * n)
        dist.all_gather_into_tensor(gathered, part)
        merged = [float(gathered[(ch * world // n) * n + ch]) for ch in range(n)]
        out["merge_sources_ok"] = merged == [float(ch) for ch in range(n)]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get() for _ in range(world))
    for r in range(world):
        assert res[r]["plans_equal"] and res[r]["covered"] and res[r]["merge_sources_ok"], res[r]
        assert res[r]["balance"] < 1.05, res[r]
