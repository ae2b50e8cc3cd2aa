"""GPU parity: the CUDA path (through the C ABI) against the f64 oracle on the same
seeded inputs.  Tolerances (north star, R20): row-infinity-relative error
per (target, layer) <= 1e-4 on the fp32 path and <= 2e-2 on the bf16 path; all
offset / indexing work exact (checked through bit-exact invariances)."""
import numpy as np
import pytest

import oracle
import workload
from _util import make_cfg, rowrel, run_gpu

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "bf16": 2e-2}


def check(wl, Z, z, tol, nthreads=8, **kw):
    Zr, zr, rows = oracle.forward_workload(wl, nthreads=nthreads, **kw)
    eZ = rowrel(Z[rows], Zr)
    assert np.isfinite(Z[rows]).all()
    assert eZ.max() <= tol, (eZ.max(), np.unravel_index(eZ.argmax(), eZ.shape))
    if z is not None:
        ez = rowrel(z[rows], zr)
        assert ez.max() <= tol, ez.max()
    return eZ.max()


def test_tiny_fp32():
    wl = workload.make_workload("tiny", seed=0)
    Z, z = run_gpu(wl)
    check(wl, Z, z, TOL["fp32"])


RAGGED = dict(lengths=np.array([1, 64, 200, 4097, 5000, 130, 9000]), m=[3, 0, 16, 64, 2, 33, 5])


def ragged_workload(dtype, d=128, h=4, M=4, L_infer=4500, seed=1, ln_affine=True, wq_scale=1.0, m=None):
    lengths = RAGGED["lengths"]
    cfg = make_cfg(B=len(lengths), d=d, h=h, M=M, dtype=dtype, L_infer=L_infer)
    wl = workload.make_workload(cfg, seed=seed, lengths=lengths, ln_affine=ln_affine, wq_scale=wq_scale)
    # ragged target counts (m_b = 0 allowed)
    m = np.array(RAGGED["m"] if m is None else m, dtype=np.int64)
    wl.tgt_off = np.concatenate([[0], np.cumsum(m)]).astype(np.int64)
    wl.xt = wl.xt[: wl.tgt_off[-1]] if wl.xt.shape[0] >= wl.tgt_off[-1] else np.resize(wl.xt, (wl.tgt_off[-1], d))
    rng = np.random.default_rng(seed + 100)
    xt = rng.standard_normal((int(wl.tgt_off[-1]), d), dtype=np.float32)
    if dtype == "bf16":
        wl.xt_bits = workload.bf16_bits(xt).reshape(xt.shape)
        wl.xt = workload.bits_to_f32(wl.xt_bits).reshape(xt.shape)
    else:
        wl.xt = xt
    return wl


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_ragged_multichunk_suffix(dtype):
    wl = ragged_workload(dtype)
    Z, z = run_gpu(wl)
    check(wl, Z, z, TOL[dtype])


def test_ragged_many_chunks_bf16():
    """chunk_keys = 1280: the 9000-key history splits into 8 chunks (the cap C <= 8), 4097 / 5000 into 4;
    split-K partials and the LSE merge on every multi-chunk request."""
    wl = ragged_workload("bf16")
    Z, z = run_gpu(wl, chunk_keys=1280)
    check(wl, Z, z, TOL["bf16"])


@pytest.mark.parametrize("d,h", [(64, 2), (256, 8)])
def test_bf16_other_widths(d, h):
    wl = ragged_workload("bf16", d=d, h=h, M=3, L_infer=0)
    Z, z = run_gpu(wl)
    check(wl, Z, z, TOL["bf16"])


def test_bf16_sharp_softmax():
    """W_Q x 8 ("sharp" regime of SURVEY §8(c)): still inside the 2e-2 bound."""
    wl = ragged_workload("bf16", wq_scale=8.0)
    Z, z = run_gpu(wl)
    check(wl, Z, z, TOL["bf16"])


@pytest.mark.parametrize("d,h", [(256, 8), (512, 8)])
def test_bf16_wide_sharp_softmax(d, h):
    """Wide kernel (d = 256 / 512, one-pass softmax with a lazy reference maximum) in the sharp
    regime, where later key tiles raise a row's maximum by more than 2^8 and O is rescaled in TMEM."""
    wl = ragged_workload("bf16", d=d, h=h, M=2, L_infer=0, wq_scale=8.0)
    Z, z = run_gpu(wl)
    check(wl, Z, z, TOL["bf16"])


# at most 16 targets x 4 heads = 64 query rows per request: the transposed (keys = MMA rows) kernel
NARROW_M = [3, 0, 16, 8, 2, 1, 5]


@pytest.mark.parametrize("chunk_keys,wq_scale", [(0, 1.0), (1280, 1.0), (0, 8.0)])
def test_bf16_narrow_requests(chunk_keys, wq_scale):
    """Requests with m_b h <= 64 (tc_attn_narrow.cu): ragged lengths 1..9000, single- and multi-chunk
    (partials + merge), and the sharp regime that triggers the lazy-maximum rescale of O^T."""
    wl = ragged_workload("bf16", m=NARROW_M, wq_scale=wq_scale)
    Z, z = run_gpu(wl, chunk_keys=chunk_keys)
    check(wl, Z, z, TOL["bf16"])


def test_rlb_and_batch_invariance_bit_exact():
    """P10/P18: a request's outputs are bit-identical alone or inside any batch."""
    wl = ragged_workload("bf16")
    Z, z = run_gpu(wl)
    for b in (2, 3, 6):
        sub = workload.Workload(cfg=wl.cfg, seed=0, weights=wl.weights, lengths=wl.lengths[b:b + 1],
                                hist_off=np.array([0, wl.lengths[b]]),
                                tgt_off=np.array([0, wl.tgt_off[b + 1] - wl.tgt_off[b]]),
                                X=wl.X[wl.hist_off[b]:wl.hist_off[b + 1]], xt=wl.xt[wl.tgt_off[b]:wl.tgt_off[b + 1]],
                                X_bits=wl.X_bits[wl.hist_off[b]:wl.hist_off[b + 1]],
                                xt_bits=wl.xt_bits[wl.tgt_off[b]:wl.tgt_off[b + 1]])
        Zb, zb = run_gpu(sub)
        t0, t1 = wl.tgt_off[b], wl.tgt_off[b + 1]
        assert np.array_equal(Zb, Z[t0:t1]) and np.array_equal(zb, z[t0:t1]), b


def test_host_buffers_equal_device_buffers():
    wl = ragged_workload("bf16")
    Zd, zd = run_gpu(wl)
    Zh, zh = run_gpu(wl, host=True)
    assert np.array_equal(Zd, Zh) and np.array_equal(zd, zh)


def test_host_input_pipelined_bit_exact():
    """Host X large enough to be streamed up in several pieces (copy stream overlapping the projection,
    include/stca.h): outputs bit-identical to device-resident inputs; the suffix-gather variant too."""
    for L_infer in (0, 7000):
        cfg = make_cfg(B=24, m=8, L_infer=L_infer)
        wl = workload.make_workload(cfg, seed=9, lengths=np.array([10000, 9999, 1, 8191] * 6))
        Zd, zd = run_gpu(wl)
        Zh, zh = run_gpu(wl, host=True)
        assert np.array_equal(Zd, Zh) and np.array_equal(zd, zh), L_infer


def test_single_key_history_exact_weight():
    """P4: L_b = 1 -> alpha = 1: the attention output is the (bf16) X~ row itself, so o is
    independent of the query; two different targets give identical Z."""
    cfg = make_cfg(B=1, m=2, dtype="bf16", M=1)
    wl = workload.make_workload(cfg, seed=4, lengths=np.array([1]))
    Z, z = run_gpu(wl)
    assert np.array_equal(Z[0, 0], Z[1, 0])
    check(wl, Z, z, TOL["bf16"])


def test_errors_leave_outputs_untouched():
    import torch
    import paper_2511_06077_b200 as stca
    wl = ragged_workload("bf16")
    c = wl.cfg
    m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer)
    X = torch.from_numpy(wl.X_bits.view(np.int16)).cuda()
    bad = wl.hist_off.copy()
    bad[2] = bad[1]  # request 1 empty
    with pytest.raises(stca.StcaError) as e:
        m.project_history(X, bad)
    assert e.value.status == -4 and "1" in e.value.message
    with pytest.raises(stca.StcaError) as e:
        m.forward(torch.zeros(3, c.d, dtype=torch.int16, device="cuda"), [0, 3],
                  torch.zeros(3, c.M, c.d, device="cuda"))
    assert e.value.status == -6  # forward before project
    m.project_history(X, wl.hist_off)
    Z = torch.full((wl.Nt, c.M, c.d), float("nan"), device="cuda")
    xt = torch.from_numpy(wl.xt_bits.view(np.int16)).cuda()
    t = wl.tgt_off.copy()
    t[-1] += 1
    with pytest.raises(stca.StcaError) as e:
        m.forward(xt, t, Z)
    assert e.value.status == -3
    torch.cuda.synchronize()
    assert torch.isnan(Z).all()
    with pytest.raises(stca.StcaError) as e:
        stca.STCA({}, d=c.d, h=c.h, r=c.r, M=c.M)
    assert e.value.status == -2 and "missing weight" in e.value.message


@pytest.mark.parametrize("name", ["serve", "train"])
def test_full_size_sampled(name):
    """BASELINE configs at full size, in the bench's launch configuration; the oracle
    checks a deterministic sample of requests (shortest, longest, first)."""
    wl = workload.make_workload(name, seed=0)
    Z, z = run_gpu(wl)
    L = wl.lengths
    sample = sorted({0, int(np.argmin(L)), int(np.argmax(L))})
    check(wl, Z, z, TOL["bf16"], requests=sample)
    assert np.isfinite(Z).all() and np.isfinite(z).all()


def _run_bits(wl, chunk_keys=0):
    """run_gpu for a bits_only workload (the multi-GB full-size configs): device inputs from the bits."""
    import torch
    import paper_2511_06077_b200 as stca
    c = wl.cfg
    m = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, L_infer=c.L_infer, dtype=c.dtype,
                  with_z=c.with_z, chunk_keys=chunk_keys)
    X = torch.from_numpy(wl.X_bits.view(np.int16)).cuda()
    xt = torch.from_numpy(wl.xt_bits.view(np.int16)).cuda()
    Z = torch.full((wl.Nt, c.M, c.d), float("nan"), device="cuda")
    z = torch.full((wl.Nt, c.d), float("nan"), device="cuda")
    m.project_history(X, wl.hist_off)
    m.forward(xt, wl.tgt_off, Z, z)
    torch.cuda.synchronize()
    m.close()
    return Z, z


def _check_sample(wl, Z, z, sample, tol):
    """The oracle on the sampled requests only (requests are independent)."""
    sub = workload.subset(wl, sample)
    Zr, zr, _ = oracle.forward_workload(sub, nthreads=8)
    rows = np.concatenate([np.arange(wl.tgt_off[b], wl.tgt_off[b + 1]) for b in sample])
    Zg, zg = Z[rows].cpu().double().numpy(), z[rows].cpu().double().numpy()
    assert np.isfinite(Zg).all() and np.isfinite(zg).all()
    eZ, ez = rowrel(Zg, Zr), rowrel(zg, zr)
    assert eZ.max() <= tol, (eZ.max(), np.unravel_index(eZ.argmax(), eZ.shape))
    assert ez.max() <= tol, ez.max()
    assert not torch_isnan_any(Z) and not torch_isnan_any(z)


def torch_isnan_any(t):
    return bool(t.isnan().any())


def test_full_size_multi_sampled():
    """The multi config at full size (8192 requests, ragged avg 2k / max 10k, m = 8: the transposed
    narrow kernel), in the bench's single-GPU launch configuration; oracle on shortest, longest, first
    and median-length requests."""
    wl = workload.make_workload("multi", seed=0, bits_only=True)
    Z, z = _run_bits(wl)
    L = wl.lengths
    sample = sorted({0, int(np.argmin(L)), int(np.argmax(L)), int(np.argsort(L)[len(L) // 2])})
    _check_sample(wl, Z, z, sample, TOL["bf16"])


def test_full_size_capacity_sampled():
    """The capacity config at full size (512 requests, d = 512, h = 8, M = 8, m = 32: the wide kernel and
    the 2-GEMM projection), bench launch configuration; the f64 oracle checks the shortest request, the
    one closest to 1000 keys and the first request whose history is at most 2000 keys (a 10k d = 512
    history costs the scalar oracle minutes; long histories are covered at this shape by
    test_capacity_shape_d512_sampled)."""
    wl = workload.make_workload("capacity", seed=0, bits_only=True)
    Z, z = _run_bits(wl)
    L = wl.lengths
    sample = sorted({int(np.argmin(L)), int(np.argmin(np.abs(L - 1000))), int(np.nonzero(L <= 2000)[0][0])})
    _check_sample(wl, Z, z, sample, TOL["bf16"])


def test_persistent_attention_more_than_128_items_per_cta():
    """k_tc_attention caches a CTA's first AT_MAXI = 128 work items in shared memory and reads later ones
    from global memory: 19200 single-tile requests with m_b h = 68 query rows (the 128-row kernel) give
    every CTA of the 148-CTA grid about 130 items; the sample covers items beyond the 128th."""
    rng = np.random.default_rng(7)
    B = 19200
    lengths = rng.integers(1, 129, size=B)
    cfg = make_cfg(B=B, m=17, M=2)
    wl = workload.make_workload(cfg, seed=9, lengths=lengths)
    Z, z = _run_bits(wl)
    _check_sample(wl, Z, z, [0, 147, 18943, 18944, 19000, 19199], TOL["bf16"])


def test_capacity_shape_d512_sampled():
    """BASELINE capacity config shape (d = 512, h = 8, M = 8, 32 targets per request), a few ragged
    requests up to L = 10k: the 2-GEMM tcgen05 projection (LayerNorm over a 512-wide TMEM row) and
    the wide tcgen05 attention kernel."""
    cfg = workload.CONFIGS["capacity"]
    wl = workload.make_workload(cfg, seed=2, B=4, lengths=np.array([10000, 64, 1500, 4104]))
    Z, z = run_gpu(wl)
    check(wl, Z, z, TOL["bf16"])


@pytest.mark.parametrize("lengths,m", [([300, 1, 4000, 129], 16), ([10000, 2500], 64)])
def test_standard_form_variant(lengths, m):
    """NEXT-3 (i): the standard attention form (Eq.(12): K^r, V^r materialised per head; stca_set_attention_form)
    computes the same function as the reordered form (oracle pin P8) -- against the oracle within the bf16
    tolerance, ragged lengths incl. L = 1 and a 10k history, up to 64 targets per request."""
    import paper_2511_06077_b200 as stca
    cfg = make_cfg(B=len(lengths), m=m, M=3)
    wl = workload.make_workload(cfg, seed=21, lengths=np.asarray(lengths))
    c = wl.cfg
    mdl = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, dtype="bf16")
    mdl.set_attention_form("standard")
    Z, z = run_gpu(wl, model=mdl)
    Zr, zr, _ = oracle.forward_workload(wl, nthreads=8)
    assert rowrel(Z, Zr).max() <= 2e-2 and rowrel(z, zr).max() <= 2e-2
    mdl.set_attention_form("reordered")  # back to the default form, same handle
    Z2, _ = run_gpu(wl, model=mdl)
    assert rowrel(Z2, Zr).max() <= 2e-2


def test_standard_form_refusals():
    import paper_2511_06077_b200 as stca
    cfg = make_cfg(B=1, m=65, M=2)  # 65 targets: more than one transposed query tile
    wl = workload.make_workload(cfg, seed=22, lengths=np.asarray([50]))
    c = wl.cfg
    mdl = stca.STCA(workload.full_weights(wl), d=c.d, h=c.h, r=c.r, M=c.M, dtype="bf16")
    mdl.set_attention_form("standard")
    with pytest.raises(stca.StcaError):
        run_gpu(wl, model=mdl)
    wide = workload.make_workload(make_cfg(B=1, m=2, d=256, h=4, M=2), seed=23, lengths=np.asarray([40]))
    cw = wide.cfg
    m2 = stca.STCA(workload.full_weights(wide), d=cw.d, h=cw.h, r=cw.r, M=cw.M, dtype="bf16")
    with pytest.raises(stca.StcaError):  # d != 128
        m2.set_attention_form("standard")
