"""Split-history over NCCL (run with torchrun, one rank per GPU): every rank gets the same
inputs, owns a block of each history's key chunks, and the per-layer partials are all-gathered
through torch.distributed; rank 0 checks bit-exactness against its own unsplit run."""
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

    ms = stca.STCA(W, d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, chunk_keys=1280, device=local,
                   split_rank=rank, split_world=world, exchange=stca.nccl_exchange())
    Zs, zs = run(ms)
    m1 = stca.STCA(W, d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, chunk_keys=1280, device=local)
    Z1, z1 = run(m1)
    ok = torch.tensor([int(torch.equal(Zs, Z1) and torch.equal(zs, z1))], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("split_nccl ok" if int(ok) == 1 else "split_nccl MISMATCH", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(ok) == 1 else 1)


if __name__ == "__main__":
    main()
