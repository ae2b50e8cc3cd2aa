"""GPU parity of the input-encoding prologue (stca_encode_history, NEXT-4) against oracle/encoding.py,
bit for bit: table values are bf16 numbers whose fp32 sum of four is exact (magnitudes in
[2^-10, 2^4): exponents within 14 bits + 8 mantissa bits < 24), so the GPU's fp32 sum rounded once
to bf16 equals the oracle's f64 sum rounded once.  Then the encoded rows feed the forward."""
import numpy as np
import pytest

import workload
from oracle import encoding as enc
from _util import make_cfg, rowrel

pytestmark = pytest.mark.gpu


def _bf16_table(rng, rows, d):
    x = rng.standard_normal((rows, d)).astype(np.float32)
    x = np.sign(x) * np.clip(np.abs(x), 2.0 ** -10, 15.0)
    return workload.bf16_bits(x).reshape(rows, d)


def _case(B, d, V, A, P, NB, seed, lengths=None):
    rng = np.random.default_rng(seed)
    L = rng.integers(1, 3000, size=B) if lengths is None else np.asarray(lengths)
    hist_off = np.concatenate([[0], np.cumsum(L)]).astype(np.int64)
    T = int(hist_off[-1])
    tabs = [_bf16_table(rng, V + 1, d), _bf16_table(rng, A + 1, d), _bf16_table(rng, P, d),
            _bf16_table(rng, NB, d) if NB else None]
    vid = rng.integers(-3, V + 3, size=T).astype(np.int64)        # includes out-of-vocabulary ids
    aid = rng.integers(-1, A + 2, size=T).astype(np.int64)
    ts = rng.integers(0, 10 ** 7, size=T).astype(np.int64)
    req = rng.integers(5 * 10 ** 6, 2 * 10 ** 7, size=B).astype(np.int64)  # some deltas negative -> bucket 0
    return hist_off, tabs, vid, aid, ts, req


@pytest.mark.parametrize("B,d,NB", [(7, 128, 24), (3, 512, 0), (1, 64, 16), (300, 128, 24)])
def test_encode_bit_exact(B, d, NB):
    import torch
    import paper_2511_06077_b200 as stca
    hist_off, tabs, vid, aid, ts, req = _case(B, d, V=5000, A=6, P=4096, NB=NB, seed=B + d)
    f32 = [workload.bits_to_f32(t).reshape(t.shape) if t is not None else None for t in tabs]
    ref = enc.encode_history(f32[0], f32[1], f32[2], f32[3], vid, aid, ts, hist_off, req)
    want = workload.bf16_bits(ref.astype(np.float32)).reshape(ref.shape)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    tt = [cu(t.view(np.int16)) if t is not None else None for t in tabs]
    X = stca.encode_history(tt[0], tt[1], tt[2], cu(vid), cu(aid), cu(hist_off), tdelta=tt[3],
                            timestamp=cu(ts) if NB else None, req_time=cu(req) if NB else None)
    torch.cuda.synchronize()
    got = X.cpu().numpy().view(np.uint16)
    assert np.array_equal(got, want), int((got != want).sum())


def test_encoded_rows_feed_the_forward():
    """Encode -> project -> forward equals the oracle forward on the oracle's encoding (R20 tolerance)."""
    import torch
    import oracle
    import paper_2511_06077_b200 as stca
    cfg = make_cfg(B=3, m=8, M=2)
    hist_off, tabs, vid, aid, ts, req = _case(3, 128, V=800, A=5, P=2048, NB=20, seed=5, lengths=[700, 1, 2100])
    f32 = [workload.bits_to_f32(t).reshape(t.shape) for t in tabs]
    Xref = enc.encode_history(f32[0], f32[1], f32[2], f32[3], vid, aid, ts, hist_off, req)
    Xbits = workload.bf16_bits(Xref.astype(np.float32)).reshape(Xref.shape)
    wl = workload.make_workload(cfg, seed=6, lengths=np.array([700, 1, 2100]))
    wl.X_bits, wl.X = Xbits, workload.bits_to_f32(Xbits).reshape(Xbits.shape)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    X = stca.encode_history(*[cu(t.view(np.int16)) for t in tabs[:3]], cu(vid), cu(aid), cu(hist_off),
                            tdelta=cu(tabs[3].view(np.int16)), timestamp=cu(ts), req_time=cu(req))
    c = wl.cfg
    m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, dtype="bf16")
    xt = cu(wl.xt_bits.view(np.int16))
    Z = torch.empty(wl.Nt, c.M, c.d, device="cuda")
    z = torch.empty(wl.Nt, c.d, device="cuda")
    m.project_history(X, hist_off)
    m.forward(xt, wl.tgt_off, Z, z)
    torch.cuda.synchronize()
    Zr, zr, _ = oracle.forward_workload(wl, nthreads=4)
    assert rowrel(Z.cpu().double().numpy(), Zr).max() <= 2e-2
    assert rowrel(z.cpu().double().numpy(), zr).max() <= 2e-2
    m.close()
