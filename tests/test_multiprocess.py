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
        import bench
        wl = workload.make_workload("multi", seed=3, B=512, bits_only=True)
        cost = bench.request_cost(wl)
        plan = torch.from_numpy(stca.plan_shards(cost, world).astype(np.int64))
        # bench.py's shard extraction on this rank: requests, offsets and rows, hashed for the parent
        mine_b = bench.shard_requests(wl, world, rank)
        sh = workload.subset(wl, mine_b, with_f32=False)
        import hashlib
        out["shard"] = (mine_b.tolist(), hashlib.sha256(sh.X_bits.tobytes()).hexdigest(),
                        hashlib.sha256(sh.xt_bits.tobytes()).hexdigest(), sh.hist_off.tolist(), sh.tgt_off.tolist())
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
        ok = {k: v for k, v in res[r].items() if k != "shard"}
        assert res[r]["plans_equal"] and res[r]["covered"] and res[r]["merge_sources_ok"], ok
        assert res[r]["balance"] < 1.05, ok
    # the ranks' shards equal a single-process split bit for bit, and together cover every request once
    import hashlib
    import bench
    wl = workload.make_workload("multi", seed=3, B=512)
    seen = []
    for r in range(world):
        reqs, hx, ht, hoff, toff = res[r]["shard"]
        assert reqs == sorted(reqs)
        seen += reqs
        rows = np.concatenate([np.arange(wl.hist_off[b], wl.hist_off[b + 1]) for b in reqs])
        trows = np.concatenate([np.arange(wl.tgt_off[b], wl.tgt_off[b + 1]) for b in reqs])
        assert hashlib.sha256(np.ascontiguousarray(wl.X_bits[rows]).tobytes()).hexdigest() == hx
        assert hashlib.sha256(np.ascontiguousarray(wl.xt_bits[trows]).tobytes()).hexdigest() == ht
        assert hoff == np.concatenate([[0], np.cumsum(wl.lengths[reqs])]).tolist()
        assert toff == np.concatenate([[0], np.cumsum(np.diff(wl.tgt_off)[reqs])]).tolist()
        assert list(bench.shard_requests(wl, world, r)) == reqs
    assert sorted(seen) == list(range(len(wl.lengths)))
