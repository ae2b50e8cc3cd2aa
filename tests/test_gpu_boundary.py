"""The C-ABI contract of include/stca.h beyond the numbers: asynchrony, handle isolation, state after
a failed projection, the per-phase profiler and the working-buffer provider.

Paper hook: one projection serves any number of forwards (RLB "compute once, reuse m times",
P:L205); the serving loop needs calls that only enqueue work (SURVEY §8(b) ownership rules)."""
import time

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


def test_calls_do_not_wait_for_the_device():
    """stca.h: project_history / forward enqueue and return; a 50+ ms spin kernel already on the stream
    must not be waited for (the work list travels through the pinned staging ring)."""
    import torch
    wl = workload.make_workload(make_cfg(B=3, m=8, M=2), seed=5, lengths=np.array([700, 90, 2500]))
    c = wl.cfg
    m = _model(wl)
    X, xt = device_inputs(wl)
    Z = torch.empty(wl.Nt, c.M, c.d, device="cuda")
    z = torch.empty(wl.Nt, c.d, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(2):  # warm: buffers grown, kernels loaded
        m.project_history(X, wl.hist_off, stream=st)
        m.forward(xt, wl.tgt_off, Z, z, stream=st)
    torch.cuda.synchronize()
    Zref = Z.clone()
    t_spin = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_spin[0].record(st)
    torch.cuda._sleep(150_000_000)  # ~75 ms at 2 GHz
    t_spin[1].record(st)
    t0 = time.perf_counter()
    for _ in range(3):
        m.project_history(X, wl.hist_off, stream=st)
        m.forward(xt, wl.tgt_off, Z, z, stream=st)
    host_ms = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    spin_ms = t_spin[0].elapsed_time(t_spin[1])
    assert spin_ms > 30.0, spin_ms
    assert host_ms < 0.5 * spin_ms, (host_ms, spin_ms)
    assert torch.equal(Z, Zref)
    m.close()


@pytest.mark.parametrize("d,h", [(128, 4), (256, 8)])
def test_two_handles_two_streams_isolated(d, h):
    """Two handles with different weights and inputs, interleaved on two streams, each give exactly
    their solo results (no shared scratch: H of the query/z FFNs and of the d != 128 projection is
    per handle)."""
    import torch
    wa = workload.make_workload(make_cfg(B=2, m=8, d=d, h=h, M=2), seed=11, lengths=np.array([1500, 300]))
    wb = workload.make_workload(make_cfg(B=3, m=4, d=d, h=h, M=2), seed=12, lengths=np.array([40, 2200, 900]))
    solo = [run_gpu(wa), run_gpu(wb)]
    ma, mb = _model(wa), _model(wb)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for wl, m, s in ((wa, ma, sa), (wb, mb, sb)):
        X, xt = device_inputs(wl)
        outs.append((wl, m, s, X, xt, torch.empty(wl.Nt, wl.cfg.M, d, device="cuda"),
                     torch.empty(wl.Nt, d, device="cuda")))
    torch.cuda.synchronize()
    for _ in range(3):
        for wl, m, s, X, xt, Z, z in outs:
            m.project_history(X, wl.hist_off, stream=s)
        for wl, m, s, X, xt, Z, z in outs:
            m.forward(xt, wl.tgt_off, Z, z, stream=s)
    torch.cuda.synchronize()
    for (wl, m, s, X, xt, Z, z), (Zs, zs) in zip(outs, solo):
        assert np.array_equal(Z.cpu().numpy().astype(np.float64), Zs)
        assert np.array_equal(z.cpu().numpy().astype(np.float64), zs)
        m.close()


def test_failed_projection_leaves_no_state():
    """A projection that fails after validation (the X~ cache cannot be allocated) leaves the handle
    without a projection: forward returns STATE instead of reading a half-written plan."""
    import torch
    import paper_2511_06077_b200 as stca
    wl = workload.make_workload(make_cfg(B=2, m=4, M=2), seed=3, lengths=np.array([64, 80]))
    m = _model(wl, chunk_keys=1 << 17)
    X, xt = device_inputs(wl)
    Z = torch.empty(wl.Nt, wl.cfg.M, wl.cfg.d, device="cuda")
    m.project_history(X, wl.hist_off)
    m.forward(xt, wl.tgt_off, Z, None)
    torch.cuda.synchronize()
    B = 1 << 20  # 2^20 histories of 2^20 rows: a 1 PB cache
    off = np.arange(B + 1, dtype=np.int64) << 20
    import ctypes
    with pytest.raises(stca.StcaError) as ei:  # T = off[B] rows claimed; X is never read (allocation fails first)
        rc = stca._lib.lib().stca_project_history(m._h, ctypes.c_void_p(X.data_ptr()), int(off[-1]),
                                                  off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), B,
                                                  ctypes.c_void_p(int(torch.cuda.current_stream().cuda_stream)))
        m._check(rc)
    assert ei.value.status == -7, ei.value  # STCA_ERR_OOM
    with pytest.raises(stca.StcaError) as ei:
        m.forward(xt, wl.tgt_off, Z, None)
    assert ei.value.status == -6, ei.value  # STCA_ERR_STATE
    # the handle still works after a fresh projection
    m.project_history(X, wl.hist_off)
    m.forward(xt, wl.tgt_off, Z, None)
    torch.cuda.synchronize()
    m.close()


@pytest.mark.parametrize("allocator", ["torch", "cuda"])
def test_profiler_regions_and_allocators(allocator):
    """stca_profile: one projection region, M attention regions per forward, one forward region; the
    results do not depend on the working-buffer provider."""
    import torch
    wl = workload.make_workload(make_cfg(B=3, m=16, M=3), seed=8, lengths=np.array([9000, 100, 3000]))
    ref = run_gpu(wl)
    m = _model(wl, allocator=allocator)
    m.profile(m.PROF_EVENTS | m.PROF_EVENTS_TARGET)
    Z, z = run_gpu(wl, model=m)
    p = m.profile_read()
    assert p["project"][1] == 1 and p["forward"][1] == 1, p
    assert p["attention"][1] == wl.cfg.M and p["merge"][1] == wl.cfg.M, p  # the 9000-key history is split
    assert p["target"][1] >= wl.cfg.M, p  # fused chain: M + 1 launches; separate GEMMs: more
    m.profile(True)  # without target regions
    run_gpu(wl, model=m)
    p = m.profile_read()
    assert p["target"][1] == 0 and p["attention"][1] == wl.cfg.M, p
    assert all(v[0] > 0 for k, v in p.items() if v[1]), p
    assert p["forward"][0] >= p["attention"][0], p
    assert np.array_equal(Z, ref[0]) and np.array_equal(z, ref[1])
    m.profile(False)
    run_gpu(wl, model=m)
    assert all(v[1] == 0 for v in m.profile_read().values())
    m.close()
    torch.cuda.synchronize()
