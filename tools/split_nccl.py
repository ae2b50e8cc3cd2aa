"""Split-history across processes (run with torchrun, one rank per GPU): every rank gets the same
inputs, owns a block of each history's key chunks; the per-layer partials are all-gathered through
torch.distributed (default) or, with --peer, read in place over peer memory (stca_split_peer_*, CUDA IPC
handles exchanged once); rank 0 checks bit-exactness against its own unsplit run."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2511_06077_b200 as stca  # noqa: E402
import workload  # noqa: E402
from _util import device_inputs, make_cfg  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = make_cfg(B=3, m=64, dtype="bf16", L_infer=10000)
    wl = workload.make_workload(cfg, seed=7, lengths=np.array([10000, 700, 3000]))
    W = workload.full_weights(wl)
    c = wl.cfg
    X, xt = device_inputs(wl)

    def run(m):
        Z = torch.full((wl.Nt, c.M, c.d), float("nan"), device="cuda")
        z = torch.full((wl.Nt, c.d), float("nan"), device="cuda")
        m.project_history(X, wl.hist_off)
        m.forward(xt, wl.tgt_off, Z, z)
        torch.cuda.synchronize()
        return Z, z

    peer = "--peer" in sys.argv
    ms = stca.STCA(W, d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, chunk_keys=1280, device=local,
                   split_rank=rank, split_world=world, exchange=None if peer else stca.nccl_exchange())
    if peer:  # exchange over peer memory: IPC handles once, then device-side epoch flags only
        small = stca.STCA(W, d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, chunk_keys=1280, device=local,
                          split_rank=rank, split_world=world)
        small.split_peer_setup(4096)  # a slot too small for this workload's partials: refused before any launch
        try:
            run(small)
            raise SystemExit("split_nccl: an over-capacity peer forward was not refused")
        except stca.StcaError:
            pass
        dist.barrier()
        small.close()
        ms.split_peer_setup(8 << 20)
    Zs, zs = run(ms)
    Zs2, zs2 = run(ms)  # second forward: the other slot, and the reuse wait
    same2 = torch.equal(Zs, Zs2) and torch.equal(zs, zs2)
    m1 = stca.STCA(W, d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, chunk_keys=1280, device=local)
    Z1, z1 = run(m1)
    ok = torch.tensor([int(torch.equal(Zs, Z1) and torch.equal(zs, z1) and same2)], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("split_nccl ok" if int(ok) == 1 else "split_nccl MISMATCH", flush=True)
    dist.barrier()  # every rank is done with the peer buffers before any handle is destroyed
    ms.close()
    dist.destroy_process_group()
    sys.exit(0 if int(ok) == 1 else 1)


if __name__ == "__main__":
    main()
