"""Stage-isolated numerics of the tcgen05 kernels against plain PyTorch fp32 references
of the same op, fed the same bf16 operands (so the only differences are accumulation
order and the output rounding)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2511_06077_b200 import _lib as L
    lib = L.lib()
    f = lib.stca_debug_tc_gemm
    f.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                  ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                  ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p]
    f.restype = ctypes.c_int
    return f


def _gemm(epi, A, Bt, Cs=None, Cf=None, g=None, b=None, eps=1e-5):
    import torch
    f = _lib()
    M, K = A.shape
    N = Bt.shape[0]
    rc = f(epi, A.data_ptr(), A.stride(0), Bt.data_ptr(), M, N, K,
           Cs.data_ptr() if Cs is not None else None, Cs.stride(0) if Cs is not None else 0,
           Cf.data_ptr() if Cf is not None else None, Cf.stride(0) if Cf is not None else 0,
           g.data_ptr() if g is not None else None, b.data_ptr() if b is not None else None, eps,
           torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc
    torch.cuda.synchronize()


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (300, 128, 128), (1000, 512, 128), (257, 128, 512),
                                   (4096, 256, 640), (77, 64, 128), (129, 32, 192)])
def test_tc_gemm_store(M, N, K):
    import torch
    torch.manual_seed(0)
    A = torch.randn(M, K, device="cuda").bfloat16()
    Bt = torch.randn(N, K, device="cuda").bfloat16()
    Cf = torch.full((M, N), float("nan"), device="cuda")
    Cs = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    _gemm(0, A, Bt, Cs=Cs, Cf=Cf)
    ref = A.float() @ Bt.float().T
    err = (Cf - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err
    assert (Cs.float() - ref).abs().max().item() / ref.abs().max().item() < 1e-2


@pytest.mark.parametrize("M,d,rd", [(300, 128, 512), (128, 64, 256), (513, 256, 1024),
                                    (40000, 512, 2048)])  # BN = 512: one accumulator, clusters loop
def test_tc_gemm_swiglu_and_ln(M, d, rd):
    import torch
    torch.manual_seed(1)
    x = torch.randn(M, d, device="cuda").bfloat16()
    Wu = (torch.rand(d, rd, device="cuda") * 2 - 1) / d ** 0.5
    Wv = (torch.rand(d, rd, device="cuda") * 2 - 1) / d ** 0.5
    Wo = (torch.rand(rd, d, device="cuda") * 2 - 1) / rd ** 0.5
    Wu, Wv, Wo = Wu.bfloat16(), Wv.bfloat16(), Wo.bfloat16()
    # chunk-interleaved W1^T: rows 64c..64c+31 = Wu[:, 32c..]^T, 64c+32.. = Wv[:, 32c..]^T
    W1t = torch.empty(2 * rd, d, device="cuda", dtype=torch.bfloat16)
    for c in range(rd // 32):
        W1t[64 * c:64 * c + 32] = Wu[:, 32 * c:32 * c + 32].T
        W1t[64 * c + 32:64 * c + 64] = Wv[:, 32 * c:32 * c + 32].T
    H = torch.zeros(M, rd, device="cuda", dtype=torch.bfloat16)
    _gemm(1, x, W1t.contiguous(), Cs=H)
    Href = (x.float() @ Wu.float()) * torch.nn.functional.silu(x.float() @ Wv.float())
    assert (H.float() - Href).abs().max().item() / Href.abs().max().item() < 1e-2
    g = 1 + 0.1 * torch.randn(d, device="cuda")
    b = 0.1 * torch.randn(d, device="cuda")
    out = torch.zeros(M, d, device="cuda", dtype=torch.bfloat16)
    outf = torch.zeros(M, d, device="cuda")
    _gemm(2, H, Wo.T.contiguous(), Cs=out, Cf=outf, g=g, b=b)
    ref = torch.nn.functional.layer_norm(H.float() @ Wo.float(), (d,), g, b, eps=1e-5)
    assert (outf - ref).abs().max().item() < 1e-3
    assert (out.float() - ref).abs().max().item() < 3e-2


@pytest.mark.parametrize("d", [128, 512])
def test_tc_gemm_ln_offset_rows(d):
    """LayerNorm epilogue on rows whose mean is ~100x their spread (the statistics are one pass of
    sums shifted by the row's first value, then the two column halves are combined): the result must
    still match a two-pass fp32 LayerNorm of the same fp32 accumulator."""
    import torch
    torch.manual_seed(3)
    M, K = 1000, 256
    A = torch.randn(M, K, device="cuda").bfloat16()
    base = torch.randn(K, device="cuda")
    Bt = (base[None, :] + 0.01 * torch.randn(d, K, device="cuda")).bfloat16()
    g = 1 + 0.1 * torch.randn(d, device="cuda")
    b = 0.1 * torch.randn(d, device="cuda")
    outf = torch.zeros(M, d, device="cuda")
    _gemm(2, A, Bt, Cf=outf, g=g, b=b)
    Y = A.double() @ Bt.double().T
    ref = torch.nn.functional.layer_norm(Y, (d,), g.double(), b.double(), eps=1e-5).float()
    spread = (Y - Y.mean(1, keepdim=True)).abs().mean().item() / Y.abs().mean().item()
    assert spread < 0.05, spread  # the rows really are offset-dominated
    assert (outf - ref).abs().max().item() < 2e-2
