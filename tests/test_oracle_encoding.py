"""Pins of the input-encoding oracle (oracle/encoding.py) against what SPEC / the
paper fix and against brute reasoning: SPEC S:L136-138 examples, bucket boundaries, OOV slots, the
recency position index (DESIGN.md R-N4a-c)."""
import numpy as np

from oracle import encoding as enc


def _tables(rng, d=8, V=5, A=3, P=4, NB=6, zero=False):
    f = (lambda *s: np.zeros(s)) if zero else (lambda *s: rng.standard_normal(s))
    return f(V + 1, d), f(A + 1, d), f(P, d), f(NB, d)


def test_zero_tables_give_zero_matrix():  # SPEC S:L136 example 1
    rng = np.random.default_rng(0)
    v, a, p, t = _tables(rng, zero=True)
    X = enc.encode_history(v, a, p, t, [1, 2, 3], [0, 1, 2], [0, 5, 9], [0, 3], [100])
    assert np.array_equal(X, np.zeros((3, 8)))


def test_single_element_is_sum_of_components():  # SPEC S:L137 example 2 (L = 1: position 0)
    rng = np.random.default_rng(1)
    v, a, p, t = _tables(rng)
    X = enc.encode_history(v, a, p, t, [4], [2], [1000], [0, 1], [1000 + 3600])
    assert np.allclose(X[0], v[4] + a[2] + p[0] + t[5])  # bucket 11 clamped to NB - 1 = 5
    X = enc.encode_history(v, a, p, None, [4], [2], None, [0, 1], None)
    assert np.allclose(X[0], v[4] + a[2] + p[0])


def test_tdelta_buckets():
    assert enc.tdelta_bucket(3600, 64) == 11  # 2^11 <= 3600 < 2^12
    for k in range(0, 40):
        assert enc.tdelta_bucket(2 ** k, 64) == k
        assert enc.tdelta_bucket(2 ** (k + 1) - 1, 64) == k
    assert enc.tdelta_bucket(0, 64) == 0 and enc.tdelta_bucket(-7, 64) == 0
    assert enc.tdelta_bucket(2 ** 40, 12) == 11


def test_oov_and_recency_positions():
    """One-hot tables make every component readable: ids outside [0, V) use row V; the position of row
    j is last - j (0 = most recent) and saturates at the table's last row."""
    d = 32
    V, A, P = 4, 2, 3
    v = np.zeros((V + 1, d)); v[np.arange(V + 1), np.arange(V + 1)] = 1      # columns 0..4
    a = np.zeros((A + 1, d)); a[np.arange(A + 1), 8 + np.arange(A + 1)] = 1  # columns 8..10
    p = np.zeros((P, d)); p[np.arange(P), 16 + np.arange(P)] = 1             # columns 16..18
    hist_off = [0, 5, 6]
    vid = [0, -1, 3, 4, 99, 2]
    aid = [1, 2, -5, 0, 1, 7]
    X = enc.encode_history(v, a, p, None, vid, aid, None, hist_off, None)
    assert [int(np.argmax(x[0:5])) for x in X] == [0, 4, 3, 4, 4, 2]
    assert [int(np.argmax(x[8:11])) for x in X] == [1, 2, 2, 0, 1, 2]
    # request 0 has rows 0..4: recency ranks 4, 3, 2, 1, 0 -> clamped to 2, 2, 2, 1, 0; request 1: rank 0
    assert [int(np.argmax(x[16:19])) for x in X] == [2, 2, 2, 1, 0, 0]
