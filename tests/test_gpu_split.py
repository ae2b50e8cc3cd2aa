"""Split-history (PAR3, BASELINE config 5): one L = 10k history split over G ranks, one
all-gather of (max, sum, O) partials per layer, every rank folding the chunks in order.
Bit-exact against the 1-GPU run with the same chunk plan (SURVEY §8(e) rule), and within
the bf16 tolerance of the oracle."""
import os
import subprocess
import sys
import threading

import numpy as np
import pytest

import oracle
import workload
from _util import device_inputs, make_cfg, rowrel

pytestmark = pytest.mark.gpu
CHUNK = 1280


def _model(wl, **kw):
    import paper_2511_06077_b200 as stca
    c = wl.cfg
    return stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype,
                     chunk_keys=CHUNK, **kw)


def _run(m, wl, stream=None):
    import torch
    c = wl.cfg
    X, xt = device_inputs(wl)
    Z = torch.full((wl.Nt, c.M, c.d), float("nan"), device="cuda")
    z = torch.full((wl.Nt, c.d), float("nan"), device="cuda")
    m.project_history(X, wl.hist_off, stream=stream)
    m.forward(xt, wl.tgt_off, Z, z, stream=stream)
    torch.cuda.synchronize()
    return Z.cpu().numpy(), z.cpu().numpy()


def split_workload(m=64):
    cfg = make_cfg(B=3, m=m, dtype="bf16", L_infer=10000)
    return workload.make_workload(cfg, seed=7, lengths=np.array([10000, 700, 3000]))


@pytest.mark.parametrize("G,m", [(2, 64), (3, 64), (8, 64), (3, 8)])  # m = 8: 32 query rows, narrow kernel
def test_split_history_threads_bit_exact(G, m):
    """G ranks as threads on one device (ThreadExchange) == the unsplit 1-GPU run, bit for bit."""
    import torch
    import paper_2511_06077_b200 as stca
    wl = split_workload(m)
    Z1, z1 = _run(_model(wl), wl)
    ex = stca.ThreadExchange(G)
    outs = [None] * G
    models = [_model(wl, split_rank=g, split_world=G, exchange=ex.for_rank(g)) for g in range(G)]

    def rank(g):
        st = torch.cuda.Stream()
        outs[g] = _run(models[g], wl, stream=st)

    th = [threading.Thread(target=rank, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
    for g in range(G):
        assert np.array_equal(outs[g][0], Z1) and np.array_equal(outs[g][1], z1), g
    Zr, zr, _ = oracle.forward_workload(wl, nthreads=8)
    assert rowrel(Z1, Zr).max() <= 2e-2 and rowrel(z1, zr).max() <= 2e-2


def test_split_peer_errors():
    import paper_2511_06077_b200 as stca
    wl = split_workload(8)
    m1 = _model(wl)
    with pytest.raises(stca.StcaError):  # not in split-history mode
        m1.split_peer_export(1 << 20)
    a, b = _model(wl, split_rank=0, split_world=2), _model(wl, split_rank=1, split_world=2)
    with pytest.raises(stca.StcaError):  # attach before export
        a.split_peer_attach([0, 0])
    ba, bb = a.split_peer_export(4096)[0], b.split_peer_export(4096)[0]
    with pytest.raises(stca.StcaError):  # own buffer not at bases[rank]
        a.split_peer_attach([bb, ba])
    with pytest.raises(stca.StcaError):  # both ranks on one device: refused (they would wait inside one GPU)
        a.split_peer_attach([ba, bb])


@pytest.mark.skipif("not __import__('torch').cuda.is_available() or __import__('torch').cuda.device_count() < 2")
def test_split_history_peer_two_gpus():
    """Peer memory across processes (CUDA IPC handles exchanged once at setup, NVLink reads), 2 GPUs."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29534", os.path.join(root, "tools", "split_nccl.py"),
                        "--peer"], capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "split_nccl ok" in r.stdout


@pytest.mark.skipif("not __import__('torch').cuda.is_available() or __import__('torch').cuda.device_count() < 2")
def test_split_history_nccl_two_gpus():
    """The same over NCCL on 2 GPUs (torchrun, one process per GPU)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(root, "tools", "split_nccl.py")],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "split_nccl ok" in r.stdout
