"""Oracle of the training data path into the ragged forward.

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module; the product path (paper_2511_06077_b200) never does.  It shares no code with the CUDA
path.  Plain Python loops over the B sequences, numpy slicing for the token copy.

Steps, in the paper's order (§3.3 "Subsequence selection" and "Batch-Level Load Balancing"):

1. train_lengths  -- Eq.(beta-scale) P:L255-258 and the rounding sentence P:L260: L_raw = L_min +
   s (L_max - L_min), rounded to the nearest multiple of 8.  s ~ Beta(alpha, beta) is drawn by the
   caller and passed in (reading R-N2a); beta_shape() is Eq.(beta) P:L266-269.
2. requested      -- the temporal suffix: request b keeps min(L_train_b, n_b) of its n_b rows.
3. allocate       -- "Global Length Allocation" P:L286 against the budget B * L_avg.  The paper gives
   no algorithm; the reading (DESIGN.md R-N2b, after SPEC's allocation design decision) is exact
   integer proportional scaling floored to multiples of 8, a floor of min(req_b, 8), then one +8 per
   sequence to the most-truncated sequences (ties: lowest index) while the slack allows.
4. compact        -- "Sequence Compaction" P:L287: the kept suffixes packed back to back into physical
   rows of exactly L_avg tokens, a sequence split across adjacent rows where needed (greedy first-fit
   in input order, SPEC's packing rule); the segment map holds (row, start, len) triples per sequence
   and the ragged index is the exclusive prefix sum of the allocated lengths.
"""
from __future__ import annotations

import math

import numpy as np


def beta_shape(alpha: float, L_min: float, L_max: float, L_avg: float) -> float:
    """Eq.(beta): beta = alpha (L_max - L_avg) / (L_avg - L_min)."""
    return alpha * (L_max - L_avg) / (L_avg - L_min)


def train_lengths(s, L_min: int, L_max: int) -> np.ndarray:
    """Eq.(beta-scale) P:L258 + P:L260.  fp64; 'nearest multiple of 8' with ties rounded up
    (reading R-N2a): L = 8 * floor(L_raw / 8 + 1/2)."""
    out = np.empty(len(s), dtype=np.int64)
    for b, sb in enumerate(s):
        L_raw = float(L_min) + float(sb) * (float(L_max) - float(L_min))
        out[b] = 8 * int(math.floor(L_raw / 8.0 + 0.5))
    return out


def requested(L_train, hist_off) -> np.ndarray:
    """keep the most recent min(L_train_b, n_b) rows of request b (n_b = its history length)."""
    B = len(L_train)
    return np.array([min(int(L_train[b]), int(hist_off[b + 1]) - int(hist_off[b])) for b in range(B)],
                    dtype=np.int64)


class InfeasibleBudget(ValueError):
    pass


def allocate(req, budget: int) -> np.ndarray:
    """Global length allocation P:L286, reading R-N2b.  Exact integers throughout."""
    req = [int(v) for v in req]
    B = len(req)
    total = sum(req)
    if total <= budget:
        return np.array(req, dtype=np.int64)
    alloc = []
    for b in range(B):
        a = 8 * ((req[b] * budget) // (8 * total))   # floor8(req_b * budget / total)
        a = max(a, min(req[b], 8))                   # every non-empty sequence keeps >= 1 row
        alloc.append(a)
    slack = budget - sum(alloc)
    if slack < 0:
        raise InfeasibleBudget(f"budget {budget} below the per-sequence floor {sum(alloc)}")
    order = sorted(range(B), key=lambda b: (-(req[b] - alloc[b]), b))
    for b in order:
        if slack < 8:
            break
        if alloc[b] + 8 <= req[b]:
            alloc[b] += 8
            slack -= 8
    return np.array(alloc, dtype=np.int64)


def compact(X, hist_off, alloc, L_avg: int):
    """Sequence compaction P:L287 (+ ragged index P:L289).

    X [T x d] (any dtype; rows are copied, never changed), hist_off [B+1], alloc [B].
    Returns (P, new_off, seg_off, segs): P [sum(alloc) x d] -- the physical rows of L_avg tokens laid
    end to end (row k = P[k L_avg : (k+1) L_avg]); new_off [B+1] the ragged index over P; segs the
    (row, start, len) triples of every sequence in order, those of sequence b at seg_off[b]..seg_off[b+1].
    """
    B = len(alloc)
    total = int(sum(int(a) for a in alloc))
    P = np.zeros((total, X.shape[1]), dtype=X.dtype)
    new_off = np.zeros(B + 1, dtype=np.int64)
    segs, seg_off = [], [0]
    pos = 0
    for b in range(B):
        a = int(alloc[b])
        src = int(hist_off[b + 1]) - a               # temporal suffix: the last a rows
        P[pos:pos + a] = X[src:src + a]
        j = 0
        while j < a:                                 # split at physical row boundaries
            row, start = (pos + j) // L_avg, (pos + j) % L_avg
            n = min(a - j, L_avg - start)
            segs.append((row, start, n))
            j += n
        pos += a
        new_off[b + 1] = pos
        seg_off.append(len(segs))
    return P, new_off, np.array(seg_off, dtype=np.int64), np.array(segs, dtype=np.int64).reshape(-1, 3)


def unpack(P, new_off):
    """Inverse view: sequence b = P[new_off[b]:new_off[b+1]] (for the round-trip pin)."""
    return [P[int(new_off[b]):int(new_off[b + 1])] for b in range(len(new_off) - 1)]
