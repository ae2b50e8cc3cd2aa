"""Time the tcgen05 GEMM (debug hook) against torch.matmul (cuBLAS) on the serve target-side shapes."""
import ctypes, sys
import torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from test_gpu_kernels import _lib
f = _lib()
st = torch.cuda.current_stream().cuda_stream
def ours(epi, A, Bt, Cs, Cf):
    M, K = A.shape; N = Bt.shape[0]
    return f(epi, A.data_ptr(), A.stride(0), Bt.data_ptr(), M, N, K, Cs.data_ptr() if Cs is not None else None,
             Cs.stride(0) if Cs is not None else 0, Cf.data_ptr() if Cf is not None else None,
             Cf.stride(0) if Cf is not None else 0, None, None, 1e-5, st)
def timeit(fn, n=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1000
M = 16384
for (N, K, epi) in [(512, 128, 0), (128, 512, 0), (128, 256, 0), (1024, 128, 1), (128, 640, 0)]:
    A = torch.randn(M, K, device='cuda').to(torch.bfloat16)
    Bt = torch.randn(N, K, device='cuda').to(torch.bfloat16)
    Cs = torch.empty(M, N // (2 if epi == 1 else 1), device='cuda', dtype=torch.bfloat16)
    t1 = timeit(lambda: ours(epi, A, Bt, Cs, None))
    t2 = timeit(lambda: torch.matmul(A, Bt.t()))
    fl = 2 * M * N * K
    print(f'M={M} N={N} K={K} epi={epi}: ours {t1:7.1f} us ({fl/t1/1e6:6.0f} TF/s)  cuBLAS {t2:7.1f} us ({fl/t2/1e6:6.0f} TF/s)')
