"""CPU tests of the C-ABI library's host side: it loads, exports every symbol
include/stca.h declares, and its exact integer work (validation, suffix truncation,
split-K chunking, attention work list, LPT shard plan) matches independent
references bit for bit.  No GPU needed: no compute calls."""
import heapq
import os
import re

import numpy as np
import pytest

import oracle
import paper_2511_06077_b200 as stca
from paper_2511_06077_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "stca.h")).read()
    declared = set(re.findall(r"\b(stca_[a-z_]+)\s*\(", hdr))
    declared.discard("stca_exchange_fn")
    assert {"stca_create", "stca_project_history", "stca_forward", "stca_destroy"} <= declared
    L = _lib.lib()
    for s in sorted(declared):
        assert hasattr(L, s), s
    assert set(_lib.SYMBOLS) == declared
    assert L.stca_abi_version() == 2


def test_status_strings():
    assert stca.status_string(0) == "STCA_OK"
    assert stca.status_string(-4) == "STCA_ERR_EMPTY_HISTORY"


def random_offsets(rng, B, maxlen, allow_empty=True):
    lo = 0 if allow_empty else 1
    L = rng.integers(lo, maxlen + 1, size=B)
    off = np.zeros(B + 1, dtype=np.int64)
    np.cumsum(L, out=off[1:])
    return off


def test_validation_matches_oracle():
    rng = np.random.default_rng(0)
    cfg = oracle._Cfg(32, 4, 2, 2, 0, 1e-5, 1)
    import ctypes
    i64p = ctypes.POINTER(ctypes.c_int64)
    for trial in range(300):
        B = int(rng.integers(0, 6))
        ho = random_offsets(rng, B, 5)
        to = random_offsets(rng, B, 3)
        T, Nt = int(ho[-1]), int(to[-1])
        kind = trial % 5
        if kind == 1 and B > 0:
            ho[rng.integers(1, B + 1)] -= 7
        elif kind == 2:
            T += 1
        elif kind == 3 and B > 0:
            to[0] = 1
        rc, bad = stca.validate_offsets(ho, to, T, Nt)
        bad_o = ctypes.c_int64(-1)
        rc_o = oracle.lib().oracle_validate(ctypes.byref(cfg), ho.ctypes.data_as(i64p), to.ctypes.data_as(i64p),
                                            B, T, Nt, ctypes.byref(bad_o))
        assert (rc, bad) == (rc_o, bad_o.value), (ho, to, T, Nt)


def test_suffix_matches_oracle_bit_exact():
    rng = np.random.default_rng(1)
    for _ in range(200):
        B = int(rng.integers(1, 20))
        ho = random_offsets(rng, B, 300)
        Li = int(rng.integers(0, 200))
        assert np.array_equal(stca.plan_suffix(ho, Li), oracle.suffix_starts(ho, Li))


@pytest.mark.parametrize("cap", [0, 128, 1280, 4096])
def test_chunks_partition(cap):
    for L in [1, 2, 127, 128, 129, 1000, 4095, 4096, 4097, 8192, 8193, 10000, 12345, 40000]:
        n, cl = stca.plan_chunks(L, cap)
        capv = cap or 8192
        assert cl % 128 == 0 and cl > 0
        assert (n - 1) * cl < L <= n * cl                      # every chunk non-empty, union = [0, L)
        assert cl <= capv or n == 1 or cl <= ((capv + 127) // 128) * 128


def test_attention_work_list_covers_exactly_once():
    rng = np.random.default_rng(2)
    for h, qtile in [(4, 128), (4, 16), (8, 128), (1, 16)]:
        B = 40
        L = rng.integers(1, 12000, size=B)
        m = rng.integers(0, 70, size=B)
        to = np.zeros(B + 1, dtype=np.int64)
        np.cumsum(m, out=to[1:])
        items = stca.plan_attention(L, to, h, qtile)
        assert np.all(np.diff(items[:, 4]) <= 0)               # LPT: key span non-increasing
        cover = {}
        for b, q0, nq, k0, kl, c in items:
            assert 1 <= nq <= qtile and kl >= 1
            key = int(b)
            cover.setdefault(key, []).append((q0, nq, k0, kl))
        for b in range(B):
            rows = int(m[b]) * h
            if rows == 0:
                assert b not in cover
                continue
            grid = np.zeros((rows, int(L[b])), dtype=np.int32)
            for q0, nq, k0, kl in cover[b]:
                q0 = q0 - to[b] * h
                grid[q0:q0 + nq, k0:k0 + kl] += 1
            assert np.all(grid == 1), b


def lpt_reference(cost, P):
    """Independent LPT: descending cost (ties: lower request), least-loaded part (ties: lower part)."""
    order = sorted(range(len(cost)), key=lambda b: (-cost[b], b))
    heap = [(0, p) for p in range(P)]
    out = [0] * len(cost)
    for b in order:
        load, p = heapq.heappop(heap)
        out[b] = p
        heapq.heappush(heap, (load + cost[b], p))
    return out


def test_lpt_shards_match_reference():
    rng = np.random.default_rng(3)
    for P in (1, 2, 4, 8):
        for _ in range(20):
            cost = rng.integers(1, 50, size=int(rng.integers(1, 300)))
            got = stca.plan_shards(cost, P)
            assert got.tolist() == lpt_reference(cost.tolist(), P)
            assert set(got.tolist()) <= set(range(P))


def test_persistent_schedule_is_a_partition():
    """stca_plan_persistent: every work item exactly once, CTA c's items are those LPT put in bin c,
    in descending cost; the bins are the stca_plan_shards (LPT) assignment."""
    rng = np.random.default_rng(5)
    for n_ctas in (1, 3, 148):
        for _ in range(10):
            cost = rng.integers(1, 40, size=int(rng.integers(1, 2000)))
            off, lst, bins = stca.plan_persistent(cost, n_ctas)
            assert off[0] == 0 and off[-1] == len(cost) and np.all(np.diff(off) >= 0)
            assert sorted(lst.tolist()) == list(range(len(cost)))
            assert bins.tolist() == lpt_reference(cost.tolist(), n_ctas)
            for c in range(n_ctas):
                mine = lst[off[c]:off[c + 1]]
                assert np.all(bins[mine] == c)
                assert np.all(np.diff(cost[mine]) <= 0)


@pytest.mark.parametrize("cap", [128, 1280, 4096])
def test_split_history_ownership_partitions_keys(cap):
    """Split-history (PAR3): ranks own contiguous, disjoint, whole-chunk key ranges covering [0, L)."""
    for L in [1, 100, 1280, 1281, 4097, 10000, 12345]:
        n, cl = stca.plan_chunks(L, cap)
        for G in range(1, 10):
            pos = 0
            for g in range(G):
                o0, ol = stca.plan_split(L, cap, G, g)
                assert o0 == pos and ol >= 0
                assert o0 % cl == 0 or ol == 0
                # every owned chunk c satisfies floor(c G / C) == g (the merge kernel's owner rule)
                for c in range(o0 // cl, (o0 + ol + cl - 1) // cl if ol else o0 // cl):
                    assert (c * G) // n == g
                pos += ol
            assert pos == L
