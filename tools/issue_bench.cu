// tools/issue_bench.cu -- cost of the single-thread tcgen05 issue pattern used by the fused kernels:
// batches of MMAs, tcgen05.commit, and mbarrier waits on barriers that have already completed.
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace stca::tc;

// pattern: 0 = 8 MMA only; 1 = 8 MMA + commit; 2 = 8 MMA + commit + wait(done barrier);
//          3 = 8 MMA + commit + wait + fence_after; 4 = like 3 plus 4 more MMAs + commit (G1+G2 shape)
template <int PAT>
__global__ void k_issue(int iters, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done, c1, c2;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    mbar_init(&c1, 1);
    mbar_init(&c2, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    mbar_arrive(&done);  // phase 0 of `done` completes: waits on parity 0 return immediately
    const uint32_t b = smem_u32(smem);
    constexpr uint32_t idesc = idesc_bf16(128, 128, 0);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) umma_f16_ts(tmem + 256, tmem + 128 + k * 8, sdesc_sw128(b + (k & 3) * 32, 16, 1024), idesc, k != 0);
      if (PAT >= 1) umma_commit(&c1);
      if (PAT >= 2) mbar_wait(&done, 0);
      if (PAT >= 3) tc_fence_after();
      if (PAT >= 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_f16_ts(tmem, tmem + 128 + k * 8, sdesc_sw128(b + (k & 3) * 32, 16, 1024), idesc, k != 0);
        umma_commit(&c2);
        mbar_wait(&done, 0);
        tc_fence_after();
      }
    }
    umma_commit(&c1);
    const long long t1 = clock64();
    out[0] = t1 - t0;
  }
  __syncthreads();
  tc_fence_before();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int PAT>
void run(const char *name) {
  unsigned long long *d, h;
  cudaMalloc(&d, 8);
  const int iters = 512;
  cudaFuncSetAttribute(k_issue<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_issue<PAT><<<1, 128, 64 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const int mmas = PAT >= 4 ? 12 : 8;
  printf("%-52s %7.1f cyc/iter (%d MMA N128 -> ideal %d)  %s\n", name, (double)h / iters, mmas, mmas * 64,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("8 MMA");
  run<1>("8 MMA + commit");
  run<2>("8 MMA + commit + wait(completed)");
  run<3>("8 MMA + commit + wait(completed) + fence::after");
  run<4>("[8 MMA + commit + wait + fence] + [4 MMA + commit + wait + fence]");
  return 0;
}
