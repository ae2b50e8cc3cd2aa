"""Host logic of bench.py's bounded oracle sample (cpu_baseline and the reference arm): the sample is
sized by the oracle's exact per-request f64 multiply-add count, and a capped sample's targets/s is scaled
by the cost per target of the sample over that of the whole workload."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import workload  # noqa: E402


def _cost_per_target(wl, reqs):
    c = [bench._oracle_cost(wl, b) for b in reqs]
    m = [int(wl.tgt_off[b + 1] - wl.tgt_off[b]) for b in reqs]
    return sum(c) / sum(m)


def test_oracle_cost_closed_form():
    # one request, L = 100 rows, m = 3 targets, d = 8, r = 2, M = 2:
    # M (L (3 r + 2) d^2 + m L 2 d) = 2 (100 * 8 * 64 + 3 * 100 * 16) = 2 * (51200 + 4800) = 112000
    cfg = workload.Config("t", B=1, m=3, d=8, h=2, r=2, M=2, dtype="fp32", L_fixed=100)
    wl = workload.make_workload(cfg, seed=1, lengths=np.array([100]))
    assert bench._oracle_cost(wl, 0) == 112000


def test_uncapped_sample_is_first_requests():
    wl = workload.make_workload("serve", seed=0, B=32, bits_only=True)
    sub, k, cap, scale = bench.oracle_subset(wl, budget_s=1e9)
    assert cap is None and scale == 1.0
    assert k == min(os.cpu_count() or 1, 32)
    assert np.array_equal(sub.lengths, wl.lengths[:k])


def test_capped_sample_fits_budget_and_scales_by_cost():
    wl = workload.make_workload("capacity", seed=0, bits_only=True)
    budget = 20.0
    sub, k, cap, scale = bench.oracle_subset(wl, budget_s=budget)
    assert cap is not None and 0 < scale < 1
    B = len(wl.lengths)
    reqs = [b for b in range(B) if wl.lengths[b] <= cap][:k]
    assert len(reqs) == k and np.array_equal(sub.lengths, wl.lengths[reqs])
    cores = os.cpu_count() or 1
    cost = [bench._oracle_cost(wl, b) for b in reqs]
    assert max(max(cost), sum(cost) / cores) / bench.ORACLE_MACS_PER_S <= budget
    assert np.isclose(scale, _cost_per_target(wl, reqs) / _cost_per_target(wl, range(B)))
