"""Session sharing: RLB extended across requests of the same user, PAPER.md P:L45
("can be extended to share across multiple requests for the same user/session") and P:L51.

The session cache must be invisible in the numbers: a forward over cached X~ rows equals, bit for bit,
the forward after a fresh stca_project_history of the same batch (the projection is row-wise and the
split-K chunking depends only on L'_b), while users whose (generation, kept length)
is cached are not projected again."""
import numpy as np
import pytest

import workload
from _util import device_inputs, make_cfg, run_gpu

pytestmark = pytest.mark.gpu


def _model(wl, **kw):
    import paper_2511_06077_b200 as stca
    c = wl.cfg
    return stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype,
                     with_z=c.with_z, **kw)


def _session_forward(m, wl, users, gens):
    import torch
    X, xt = device_inputs(wl)
    n = m.project_history_session(users, gens, X, wl.hist_off)
    Z = torch.full((wl.Nt, wl.cfg.M, wl.cfg.d), float("nan"), device="cuda")
    z = torch.full((wl.Nt, wl.cfg.d), float("nan"), device="cuda")
    m.forward(xt, wl.tgt_off, Z, z)
    torch.cuda.synchronize()
    return n, Z.cpu().numpy().astype(np.float64), z.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("m_t", [8, 64])  # transposed narrow kernel / 128-row kernel
def test_session_hits_equal_fresh_projection(m_t):
    base = workload.make_workload(make_cfg(B=6, m=m_t, M=3, L_infer=9000), seed=31,
                                  lengths=np.array([900, 9500, 130, 2047, 1, 4000]))
    mdl = _model(base)
    mdl.session_open(40000)
    # call 1: users 10..13 (requests 0..3), all new
    b1 = workload.subset(base, [0, 1, 2, 3])
    n, Z, z = _session_forward(mdl, b1, [10, 11, 12, 13], [1, 1, 1, 1])
    assert n == 4
    Zr, zr = run_gpu(b1)
    assert np.array_equal(Z, Zr) and np.array_equal(z, zr)
    # call 2: user 11 unchanged (hit), user 13 with a new history (request 4's rows, generation 2), user 15 new
    b2 = workload.subset(base, [1, 4, 5])
    n, Z, z = _session_forward(mdl, b2, [11, 13, 15], [1, 2, 1])
    assert n == 2
    Zr, zr = run_gpu(b2)
    assert np.array_equal(Z, Zr) and np.array_equal(z, zr)
    # call 3: the same batch again -> nothing projected, same bits
    n, Z3, z3 = _session_forward(mdl, b2, [11, 13, 15], [1, 2, 1])
    assert n == 0
    assert np.array_equal(Z3, Zr) and np.array_equal(z3, zr)
    # a user twice in one batch with the same history shares one entry
    b4 = workload.subset(base, [1, 1, 2])
    n, Z, z = _session_forward(mdl, b4, [11, 11, 12], [1, 1, 1])
    assert n == 0
    Zr, zr = run_gpu(b4)
    assert np.array_equal(Z, Zr) and np.array_equal(z, zr)
    mdl.close()


def test_session_eviction_fifo_ring():
    """Capacity 2500 rows, users of 1000 rows: the ring wraps and evicts; results stay exact."""
    base = workload.make_workload(make_cfg(B=5, m=4, M=2), seed=32, lengths=np.array([1000, 1000, 1000, 1000, 1000]))
    mdl = _model(base)
    mdl.session_open(2500)
    seq = [([0, 1], [1, 2], 2),    # u1 [0, 1000), u2 [1000, 2000)
           ([0, 1], [1, 2], 0),    # both cached
           ([2], [3], 1),          # 1000 rows at 2000 do not fit -> wrap to 0: u3 [0, 1000) evicts u1
           ([0], [1], 1),          # u1 again at [1000, 2000), evicting u2
           ([1, 2], [2, 3], 2),    # u2 at 2000 wraps onto u3, a hit of this batch -> reset, both projected
           ([3, 4], [4, 5], 2)]    # 2000 rows at 2000 wrap to 0: evict u2, u3
    for reqs, users, want in seq:
        b = workload.subset(base, reqs)
        n, Z, z = _session_forward(mdl, b, users, [1] * len(users))
        assert n == want, (reqs, n, want)
        Zr, zr = run_gpu(b)
        assert np.array_equal(Z, Zr) and np.array_equal(z, zr)
    mdl.close()


def test_session_errors():
    import paper_2511_06077_b200 as stca
    base = workload.make_workload(make_cfg(B=2, m=4, M=2), seed=33, lengths=np.array([300, 200]))
    mdl = _model(base)
    X, _ = device_inputs(base)
    with pytest.raises(stca.StcaError) as e:
        mdl.project_history_session([1, 2], [1, 1], X, base.hist_off)
    assert e.value.status == -6  # STATE: no session
    mdl.session_open(400)
    with pytest.raises(stca.StcaError) as e:
        mdl.project_history_session([1, 2], [1, 1], X, base.hist_off)
    assert e.value.status == -7  # OOM: 500 new rows > 400
    with pytest.raises(stca.StcaError) as e:
        mdl.project_history_session([1, 1], [1, 2], X, base.hist_off)
    assert e.value.status == -1  # one user, two histories
    assert mdl.project_history_session([1], [1], X[:300], base.hist_off[:2]) == 1
    mdl.close()
