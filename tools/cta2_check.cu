// tools/cta2_check.cu -- validates the CTA-pair (cta_group::2) tcgen05 path: M = 256 across a
// cluster of 2 CTAs, A rows [128 r, 128 r + 128) in CTA r's TMEM (TS) or SMEM (SS), B^T rows
// [N/2 r, N/2 (r+1)) in CTA r's SMEM, D rows of CTA r in its own TMEM; leader issues the MMA and
// commits to both CTAs' mbarriers.  Also times back-to-back M=256 MMAs.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "tc_ptx.cuh"

using namespace stca::tc;

constexpr int K = 64, N = 128;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) k_cta2(const __nv_bfloat16 *A /*[256 x K]*/, const __nv_bfloat16 *Bt /*[N x K]*/,
                                                 float *D /*[256 x N]*/, int mode, int iters, unsigned long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, row = threadIdx.x;
  const uint32_t rank = cluster_rank();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  // this CTA's half of B^T (N/2 rows) and its 128 rows of A, K-major SW128
  for (int n = threadIdx.x; n < N / 2; n += blockDim.x)
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<uint4 *>(smem + sw128_off(n, c)) =
          *reinterpret_cast<const uint4 *>(Bt + (rank * (N / 2) + n) * K + c * 8);
  for (int m = threadIdx.x; m < 128; m += blockDim.x)
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<uint4 *>(smem + 16384 + sw128_off(m, c)) =
          *reinterpret_cast<const uint4 *>(A + (rank * 128 + m) * K + c * 8);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  {
    uint32_t w[16];
    for (int blk = 0; blk < K / 32; ++blk) {
      for (int j = 0; j < 16; ++j) {
        const __nv_bfloat16 lo = A[(rank * 128 + row) * K + blk * 32 + 2 * j], hi = A[(rank * 128 + row) * K + blk * 32 + 2 * j + 1];
        w[j] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
      }
      tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + 256 + blk * 16, w);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(256, N, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int k = 0; k < K / 16; ++k) {
        const uint64_t bd = sdesc_sw128(smem_u32(smem) + k * 32, 16, 1024);
        const uint32_t acc = (it | k) != 0 && iters == 1 ? 1u : (k != 0);
        if (mode == 0) {
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
                  tmem),
              "r"(tmem + 256 + k * 8), "l"(bd), "r"(idesc), "r"(acc)
              : "memory");
        } else {
          const uint64_t ad = sdesc_sw128(smem_u32(smem) + 16384 + k * 32, 16, 1024);
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                  tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
              : "memory");
        }
      }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(&bar)),
                 "h"((unsigned short)3)
                 : "memory");
    mbar_wait(&bar, 0);
    cyc[0] = clock64() - t0;
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(rank * 128 + row) * N + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

int main() {
  static __nv_bfloat16 hA[256 * K], hB[N * K];
  static float fA[256 * K], fB[N * K], hD[256 * N];
  srand(1);
  for (int i = 0; i < 256 * K; ++i) { hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < N * K; ++i) { hB[i] = __float2bfloat16((rand() % 13 - 6) / 4.f); fB[i] = __bfloat162float(hB[i]); }
  __nv_bfloat16 *dA, *dB;
  float *dD;
  unsigned long long *dc, hc;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_cta2, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dD, 0, sizeof hD);
    k_cta2<<<2, 128, 64 * 1024>>>(dA, dB, dD, mode, 1, dc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 256; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)fA[m * K + k] * fB[n * K + k];
        maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]));
      }
    printf("cta_group::2 %s: max abs err %.3e (%s)\n", mode == 0 ? "TS" : "SS", maxerr, cudaGetErrorString(e));
    const int iters = 1024;
    k_cta2<<<2, 128, 64 * 1024>>>(dA, dB, dD, mode, iters, dc);
    e = cudaDeviceSynchronize();
    cudaMemcpy(&hc, dc, 8, cudaMemcpyDeviceToHost);
    const double per = (double)hc / (iters * (K / 16));
    printf("   timing: %.1f cyc per M256 N%d K16 MMA -> %.0f MAC/cyc per SM (%s)\n", per, N, 256.0 * N * 16 / per / 2,
           cudaGetErrorString(e));
  }
  return 0;
}
