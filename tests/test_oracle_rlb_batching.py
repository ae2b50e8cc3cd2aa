"""Pins of oracle/rlb_batching.py (NEXT-2 training data path) against what the paper and arithmetic fix.

Each case is derived by hand or by an independent brute force, never by re-calling the oracle's own
formula: PAPER.md P:L255-289, SPEC.md S:L248-265 examples.
"""
import numpy as np
import pytest

from oracle import rlb_batching as rb


def test_beta_shape_symmetric_and_mean():
    # L_avg midway between L_min and L_max -> symmetric Beta(alpha, alpha) (Eq. beta)
    assert rb.beta_shape(0.3, 0, 4096, 2048) == pytest.approx(0.3)
    # the expectation constraint P:L263: L_min + (L_max - L_min) alpha / (alpha + beta) == L_avg
    a = 0.5
    b = rb.beta_shape(a, 64, 4096, 1024)
    assert 64 + (4096 - 64) * a / (a + b) == pytest.approx(1024)
    # and by sampling (the caller's draw, seeded): the sample mean of L_raw approaches L_avg
    s = np.random.default_rng(0).beta(a, b, size=400_000)
    assert np.mean(64 + s * (4096 - 64)) == pytest.approx(1024, rel=5e-3)


def _nearest8_bruteforce(x):
    cands = [8 * k for k in range(0, int(x // 8) + 3)]
    best = min(abs(x - c) for c in cands)
    return max(c for c in cands if abs(x - c) == best)   # ties up (reading R-N2a)


def test_train_lengths_endpoints_and_rounding():
    assert list(rb.train_lengths([0.0, 1.0], 64, 4096)) == [64, 4096]
    # L_raw = 10 -> 8 ; L_raw = 12 (tie) -> 16 ; L_raw = 13 -> 16
    assert list(rb.train_lengths([0.5], 0, 20)) == [8]
    assert list(rb.train_lengths([0.5], 0, 24)) == [16]
    assert list(rb.train_lengths([0.5], 0, 26)) == [16]
    rng = np.random.default_rng(1)
    s = rng.random(2000)
    got = rb.train_lengths(s, 37, 3001)
    want = [_nearest8_bruteforce(37 + float(v) * (3001 - 37)) for v in s]
    assert list(got) == want


def test_requested_is_temporal_suffix_length():
    hist_off = np.array([0, 100, 105, 405])
    assert list(rb.requested([64, 64, 256], hist_off)) == [64, 5, 256]


def test_allocate_under_budget_identity_and_symmetric():
    assert list(rb.allocate([40, 8, 17], 100)) == [40, 8, 17]
    assert list(rb.allocate([4096, 4096], 2 * 2048)) == [2048, 2048]


def test_allocate_hand_cases():
    # (80, 16), budget 56: floor8 of 46.67 and 9.33 -> (40, 8); slack 8 to the most truncated (seq 0)
    assert list(rb.allocate([80, 16], 56)) == [48, 8]
    # (16, 16), budget 24: (8, 8), slack 8, equal truncation -> lowest index
    assert list(rb.allocate([16, 16], 24)) == [16, 8]
    # short sequence keeps min(req, 8) rows: (5, 400), budget 104 -> floor8(1.27)=0 -> 5; 8*floor(102.7/8)=96
    assert list(rb.allocate([5, 400], 104)) == [5, 96]
    with pytest.raises(rb.InfeasibleBudget):
        rb.allocate([100, 100, 100], 16)


def test_allocate_budget_invariants_seeded_sweep():
    rng = np.random.default_rng(2)
    for trial in range(3000):
        B = int(rng.integers(1, 40))
        L_avg = 8 * int(rng.integers(1, 64))
        req = rng.integers(1, 8 * L_avg, size=B)
        if trial % 2:
            req = 8 * np.maximum(req // 8, 1)                            # rounded L_train
        budget = B * L_avg
        try:
            a = rb.allocate(req, budget)
        except rb.InfeasibleBudget:
            assert req.sum() > budget            # only an over-budget batch can be infeasible
            continue
        assert a.sum() <= budget                                         # hard bound
        assert np.all(a <= req) and np.all(a >= np.minimum(req, 8))
        assert np.all((a % 8 == 0) | (a == req))
        if req.sum() > budget and trial % 2 and np.all(req >= 8):
            assert a.sum() > budget - 8                                  # slack pass exhausts the budget


def test_compact_spec_example_and_identity():
    d = 3
    X = np.arange(8 * d).reshape(8, d)
    # B=2, L_avg=4, lengths (6, 2): row0 = seq0[0..4], row1 = seq0[4..6] || seq1[0..2]
    P, off, seg_off, segs = rb.compact(X, np.array([0, 6, 8]), [6, 2], 4)
    assert np.array_equal(P, X)
    assert list(off) == [0, 6, 8] and list(seg_off) == [0, 2, 3]
    assert segs.tolist() == [[0, 0, 4], [1, 0, 2], [1, 2, 2]]
    # identity packing: every sequence exactly L_avg
    P, off, seg_off, segs = rb.compact(X, np.array([0, 4, 8]), [4, 4], 4)
    assert segs.tolist() == [[0, 0, 4], [1, 0, 4]]


def test_compact_keeps_suffix_and_round_trips():
    rng = np.random.default_rng(3)
    for _ in range(50):
        B = int(rng.integers(1, 12))
        n = rng.integers(1, 60, size=B)
        hist_off = np.concatenate([[0], np.cumsum(n)])
        X = rng.integers(0, 1 << 16, size=(int(hist_off[-1]), 5)).astype(np.uint16)
        alloc = np.array([int(rng.integers(1, v + 1)) for v in n])
        L_avg = int(rng.integers(1, 30))
        P, off, seg_off, segs = rb.compact(X, hist_off, alloc, L_avg)
        for b, part in enumerate(rb.unpack(P, off)):
            assert np.array_equal(part, X[hist_off[b + 1] - alloc[b]:hist_off[b + 1]])   # most recent rows
            tri = segs[seg_off[b]:seg_off[b + 1]]
            assert tri[:, 2].sum() == alloc[b]
            assert np.all(tri[:, 1] + tri[:, 2] <= L_avg)
            flat = tri[:, 0] * L_avg + tri[:, 1]
            assert flat[0] == off[b] and np.all(np.diff(flat) == tri[:-1, 2])
