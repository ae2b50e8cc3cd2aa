"""Oracle of the input-encoding prologue -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this module; the
product path (paper_2511_06077_b200/) never does.  Plain numpy, float64, one obvious loop per step.

PAPER.md §3.1.1 "Input encoding": "Each historical element (v_j, a_j) is embedded as
x_j in R^d (video, action-type, position fused)"; Table "Time-delta side info": "Add per-token
feature: request time minus item timestamp (recency prior)".  SPEC.md S:L130-138 (encode_history):
x_j = video_emb + action_emb + position_emb (+ time_delta_emb), unknown ids map to a reserved OOV
slot, time deltas in log2-second buckets (3600 s -> bucket 11).

Readings (DESIGN.md R-N4a..c; the paper is silent on all three):
* R-N4a position index: recency rank, p_j = (last row of the request) - j, so 0 is the most recent
  element and a position means the same thing for a 2k training window and a 10k serving history
  (the "train sparsely, infer densely" regimen); ranks beyond the table share its last row.
* R-N4b OOV: the video / action tables have one extra row (index V / A) that every id outside
  [0, V) / [0, A) uses.
* R-N4c time-delta bucket: dt = request time - timestamp in seconds; bucket = floor(log2(dt)) for
  dt >= 1 (exactly: dt.bit_length() - 1), 0 for dt < 1, clamped to the table's last row.
The sum is taken in f64 and rounded once to the storage precision (bf16 RNE for the bf16 path).
"""
from __future__ import annotations

import numpy as np


def tdelta_bucket(dt: int, n_buckets: int) -> int:
    """R-N4c: floor(log2(dt)) for dt >= 1 (integer bit length: no float rounding at powers of two)."""
    dt = int(dt)
    b = dt.bit_length() - 1 if dt >= 1 else 0
    return min(b, n_buckets - 1)


def encode_history(video, action, position, tdelta, video_id, action_id, timestamp, hist_off, req_time):
    """X [T x d] float64: x_j = video[v'_j] + action[a'_j] + position[p_j] (+ tdelta[bucket_j]).
    video [V+1 x d], action [A+1 x d] (last row = OOV), position [P x d], tdelta [NB x d] or None;
    ids / timestamps int64 [T], hist_off int64 [B+1], req_time int64 [B]."""
    video, action, position = (np.asarray(t, dtype=np.float64) for t in (video, action, position))
    V, A, P = video.shape[0] - 1, action.shape[0] - 1, position.shape[0]
    T = int(hist_off[-1])
    X = np.zeros((T, video.shape[1]), dtype=np.float64)
    for b in range(len(hist_off) - 1):
        last = int(hist_off[b + 1]) - 1
        for j in range(int(hist_off[b]), int(hist_off[b + 1])):
            v = int(video_id[j])
            a = int(action_id[j])
            v = v if 0 <= v < V else V
            a = a if 0 <= a < A else A
            p = min(last - j, P - 1)
            x = video[v] + action[a] + position[p]
            if tdelta is not None:
                td = np.asarray(tdelta, dtype=np.float64)
                x = x + td[tdelta_bucket(int(req_time[b]) - int(timestamp[j]), td.shape[0])]
            X[j] = x
    return X
