"""GPU parity of the training data path (stca_rlb_allocate / stca_rlb_compact, NEXT-2) against
oracle/rlb_batching.py on the same seeded inputs.  Integer and copy work: bit-exact everywhere.

Input recipe: full user histories n_b drawn like the multi config's (Beta
lengths on [64, 10000], mean 2000), s_b ~ Beta(alpha, beta(alpha, L_min, L_max, L_avg)) with the train
config's L_min = 64, L_max = 4096, L_avg = 2048, alpha = 0.02 (U-shaped); X bf16 rows as bits.
"""
import numpy as np
import pytest

from oracle import rlb_batching as rb
from workload import CONFIGS, sample_lengths

pytestmark = pytest.mark.gpu


def _case(seed, B, L_min, L_max, L_avg, alpha=0.02, n_max=None, d=8):
    rng = np.random.default_rng(seed)
    if n_max is None:
        n = sample_lengths(rng, CONFIGS["multi"], B)
    else:
        n = rng.integers(0, n_max + 1, size=B)
    hist_off = np.concatenate([[0], np.cumsum(n)]).astype(np.int64)
    s = rng.beta(alpha, rb.beta_shape(alpha, L_min, L_max, L_avg), size=B)
    X = rng.integers(0, 1 << 16, size=(int(hist_off[-1]), d), dtype=np.uint16)
    return s, hist_off, X


def _gpu(s, hist_off, X, L_min, L_max, L_avg):
    import torch
    import paper_2511_06077_b200 as stca
    dev = torch.device("cuda:0")
    s_d = torch.from_numpy(s).to(dev)
    off_d = torch.from_numpy(hist_off).to(dev)
    X_d = torch.from_numpy(X.view(np.int16)).to(dev)
    alloc, new_off = stca.rlb_allocate(s_d, off_d, L_min, L_max, L_avg)
    P, seg_off, segs = stca.rlb_compact(X_d, off_d, alloc, new_off, L_avg)
    torch.cuda.synchronize()
    return alloc.cpu().numpy(), new_off.cpu().numpy(), P, seg_off.cpu().numpy(), segs.cpu().numpy()


def _check(s, hist_off, X, L_min, L_max, L_avg, full_rows=True):
    want_alloc = rb.allocate(rb.requested(rb.train_lengths(s, L_min, L_max), hist_off), len(s) * L_avg)
    alloc, new_off, P, seg_off, segs = _gpu(s, hist_off, X, L_min, L_max, L_avg)
    assert np.array_equal(alloc, want_alloc)
    if full_rows:
        Pw, off_w, seg_off_w, segs_w = rb.compact(X, hist_off, want_alloc, L_avg)
        assert np.array_equal(P[:len(Pw)].cpu().numpy().view(np.uint16), Pw)
    else:   # full size: the oracle's one-row-at-a-time definition on sampled rows
        off_w = np.concatenate([[0], np.cumsum(want_alloc)])
        rng = np.random.default_rng(7)
        rows = rng.integers(0, int(off_w[-1]), size=4096)
        b = np.searchsorted(off_w, rows, side="right") - 1
        src = hist_off[b + 1] - want_alloc[b] + (rows - off_w[b])
        import torch
        got = P[torch.from_numpy(rows).to(P.device)].cpu().numpy().view(np.uint16)
        assert np.array_equal(got, X[src])
        _, _, seg_off_w, segs_w = rb.compact(np.zeros((int(hist_off[-1]), 0), np.uint16), hist_off, want_alloc, L_avg)
    assert np.array_equal(new_off, off_w)
    assert np.array_equal(seg_off, seg_off_w)
    assert np.array_equal(segs[:seg_off[-1]], segs_w)
    return alloc


@pytest.mark.parametrize("seed,B,n_max,L_min,L_max,L_avg", [
    (0, 1, 50, 8, 64, 16),          # single request
    (1, 7, 300, 16, 256, 64),       # ragged, over budget
    (2, 33, 20, 8, 64, 32),         # short histories: under budget -> alloc == req
    (3, 300, 500, 32, 512, 128),    # several warps, ragged tail
    (4, 1500, 200, 8, 256, 40),     # > 1024 requests: multi-pass scans; L_avg not a multiple of 8
    (5, 64, 1, 8, 64, 16),          # histories of 0 or 1 rows (empty ones keep nothing)
])
def test_rlb_small_parity(seed, B, n_max, L_min, L_max, L_avg):
    s, hist_off, X = _case(seed, B, L_min, L_max, L_avg, n_max=n_max, alpha=0.5)
    _check(s, hist_off, X, L_min, L_max, L_avg)


def test_rlb_train_config_full_size():
    """B = 1024 at the train config's length law, d = 128 bf16 rows (256 B), ~2M history rows."""
    import torch
    cfg = CONFIGS["train"]
    s, hist_off, X = _case(11, cfg.B, cfg.L_min, cfg.L_max, cfg.L_avg, d=cfg.d)
    alloc = _check(s, hist_off, X, cfg.L_min, cfg.L_max, cfg.L_avg, full_rows=False)
    assert alloc.sum() <= cfg.B * cfg.L_avg
    # timing of the copy (informational; DESIGN.md NEXT-2 row): read + write of sum(alloc) rows
    import paper_2511_06077_b200 as stca
    dev = torch.device("cuda:0")
    X_d = torch.from_numpy(X.view(np.int16)).to(dev)
    off_d = torch.from_numpy(hist_off).to(dev)
    a_d, n_d = stca.rlb_allocate(torch.from_numpy(s).to(dev), off_d, cfg.L_min, cfg.L_max, cfg.L_avg)
    P = torch.empty((cfg.B * cfg.L_avg, cfg.d), dtype=torch.int16, device=dev)
    for _ in range(3):
        stca.rlb_compact(X_d, off_d, a_d, n_d, cfg.L_avg, P=P)
    # each call timed alone with CUDA events, after writing a 256 MB buffer (> the 126 MB L2): cold L2
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    reps, tot = 20, 0.0
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        stca.rlb_compact(X_d, off_d, a_d, n_d, cfg.L_avg, P=P)
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    ms = tot / reps
    nbytes = 2 * int(alloc.sum()) * cfg.d * 2
    print(f"\nrlb_compact train (L2 flushed before each call): {ms * 1e3:.1f} us per call, "
          f"{nbytes / ms / 1e6:.0f} GB/s algorithmic")


def test_rlb_errors():
    import torch
    import paper_2511_06077_b200 as stca
    dev = torch.device("cuda:0")
    off = torch.tensor([0, 100, 200, 300], dtype=torch.int64, device=dev)
    with pytest.raises(stca.StcaError):    # infeasible: floors of 8 each exceed 3 * 1
        stca.rlb_allocate(torch.full((3,), 0.9, dtype=torch.float64, device=dev), off, 8, 64, 1)
    with pytest.raises(stca.StcaError):    # s outside [0, 1]
        stca.rlb_allocate(torch.tensor([0.1, 1.5, 0.2], dtype=torch.float64, device=dev), off, 8, 64, 16)
    a, n = stca.rlb_allocate(torch.full((3,), 0.5, dtype=torch.float64, device=dev), off, 8, 64, 16)
    with pytest.raises(stca.StcaError):    # rows of 6 bytes: not a multiple of 16
        stca.rlb_compact(torch.zeros((300, 3), dtype=torch.int16, device=dev), off, a, n, 16)


def test_rlb_compacted_batch_feeds_the_forward():
    """NEXT-2 end to end: the compacted rows P and their ragged index new_off go straight into
    stca_project_history / stca_forward; the result equals the oracle forward on the oracle's own
    compaction (bf16 tolerance, R20).  L_avg = 96 puts segment boundaries inside 128-row tiles."""
    import dataclasses

    import torch

    import oracle
    import paper_2511_06077_b200 as stca
    import workload
    from _util import make_cfg, rowrel

    lengths = np.array([300, 50, 1000, 7, 600, 129, 2500])
    B, L_min, L_max, L_avg = len(lengths), 8, 1024, 96
    cfg = make_cfg(B=B, m=4, d=128, h=4, M=2, dtype="bf16")
    wl = workload.make_workload(cfg, seed=5, lengths=lengths, ln_affine=True)
    # lengths drawn for a mean of 400 against a budget of 96 per request: over budget (1061 > 672 rows)
    s = np.random.default_rng(6).beta(0.5, rb.beta_shape(0.5, L_min, L_max, 400), size=B)

    want_alloc = rb.allocate(rb.requested(rb.train_lengths(s, L_min, L_max), wl.hist_off), B * L_avg)
    Pw, off_w, _, _ = rb.compact(wl.X, wl.hist_off, want_alloc, L_avg)
    Pw_bits, _, _, _ = rb.compact(wl.X_bits, wl.hist_off, want_alloc, L_avg)
    assert rb.requested(rb.train_lengths(s, L_min, L_max), wl.hist_off).sum() > B * L_avg
    wl_c = dataclasses.replace(wl, X=Pw, X_bits=Pw_bits, hist_off=off_w)
    Zr, zr, rows = oracle.forward_workload(wl_c, nthreads=8)

    dev = torch.device("cuda:0")
    off_d = torch.from_numpy(wl.hist_off).to(dev)
    X_d = torch.from_numpy(wl.X_bits.view(np.int16)).to(dev)
    alloc, new_off = stca.rlb_allocate(torch.from_numpy(s).to(dev), off_d, L_min, L_max, L_avg)
    P, _, _ = stca.rlb_compact(X_d, off_d, alloc, new_off, L_avg)
    new_off_h = new_off.cpu().numpy()
    assert np.array_equal(new_off_h, off_w)
    m = stca.STCA(workload.full_weights(wl), d=cfg.d, h=cfg.h, r=cfg.r, M=cfg.M, L_infer=0, dtype="bf16",
                  with_z=cfg.with_z)
    xt = torch.from_numpy(wl.xt_bits.view(np.int16)).to(dev)
    Z = torch.full((wl.Nt, cfg.M, cfg.d), float("nan"), dtype=torch.float32, device=dev)
    z = torch.full((wl.Nt, cfg.d), float("nan"), dtype=torch.float32, device=dev)
    m.project_history(P[:int(new_off_h[-1])].contiguous(), new_off_h)
    m.forward(xt, wl.tgt_off, Z, z)
    torch.cuda.synchronize()
    Z, z = Z.cpu().numpy().astype(np.float64), z.cpu().numpy().astype(np.float64)
    assert rowrel(Z[rows], Zr).max() <= 2e-2
    assert rowrel(z[rows], zr).max() <= 2e-2
