"""Small cases that drive every kernel of libstca once, for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run).  Checks the results against the f64 oracle so a sanitizer run also
proves the run computed the right thing.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import workload  # noqa: E402
from _util import make_cfg, rowrel, run_gpu  # noqa: E402


def case(cfg, lengths, seed, tol, **kw):
    wl = workload.make_workload(cfg, seed=seed, lengths=np.asarray(lengths))
    Z, z = run_gpu(wl, **kw)
    Zr, zr, _ = oracle.forward_workload(wl, nthreads=4)
    e = max(rowrel(Z, Zr).max(), rowrel(z, zr).max())
    print(f"{cfg.name} d={cfg.d} m={cfg.m} L={list(lengths)}: max row-inf-rel {e:.2e}", flush=True)
    assert e <= tol, e


def main():
    import torch
    import paper_2511_06077_b200 as stca
    # narrow (m h = 32 <= 64) + split-K merge (9000 > 8192 keys) + fused d = 128 projection
    case(make_cfg("narrow", B=3, m=8, M=2), [9000, 1, 300], 1, 2e-2)
    # 128-row kernel (m h = 256), a partial last query tile (m h = 132)
    case(make_cfg("regular", B=2, m=64, M=2), [700, 129], 2, 2e-2)
    case(make_cfg("regular2", B=1, m=33, M=2), [1000], 3, 2e-2)
    # wide kernel + 2-GEMM projection (d = 256)
    case(make_cfg("wide", B=2, m=16, d=256, h=8, M=2), [300, 65], 4, 2e-2)
    # fp32 CUDA-core path
    case(make_cfg("fp32", B=2, m=4, d=64, h=2, M=2, dtype="fp32"), [100, 7], 5, 1e-4)
    # training data path: allocation + compaction
    hist_off = np.array([0, 300, 350, 1350], dtype=np.int64)
    s = torch.tensor([0.9, 0.2, 0.7], dtype=torch.float64, device="cuda")
    off_d = torch.from_numpy(hist_off).cuda()
    alloc, new_off = stca.rlb_allocate(s, off_d, 8, 1024, 96)
    Xb = torch.zeros(1350, 128, dtype=torch.int16, device="cuda")
    stca.rlb_compact(Xb, off_d, alloc, new_off, 96)
    torch.cuda.synchronize()
    print("sanitize cases ok", flush=True)


if __name__ == "__main__":
    main()
