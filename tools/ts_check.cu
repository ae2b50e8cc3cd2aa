// tools/ts_check.cu -- validates the TMEM layout of a tcgen05.mma A operand (kind::f16, M = 128):
// row m in TMEM lane m, K elements packed two per 32-bit column (low half = even k).
// D = A . B^T with A written by tcgen05.st, B^T K-major SW128 in SMEM; compared on the host.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "tc_ptx.cuh"

using namespace stca::tc;

constexpr int K = 64, N = 128;

__global__ void k_ts(const __nv_bfloat16 *A /*[128 x K]*/, const __nv_bfloat16 *Bt /*[N x K]*/, float *D, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, row = threadIdx.x;
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  // B^T into SMEM, K-major SW128 (one 64-element atom column)
  for (int n = threadIdx.x; n < N; n += blockDim.x)
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<uint4 *>(smem + sw128_off(n, c)) = *reinterpret_cast<const uint4 *>(Bt + n * K + c * 8);
  // A for SS mode, same layout
  for (int m = threadIdx.x; m < 128; m += blockDim.x)
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<uint4 *>(smem + 16384 + sw128_off(m, c)) = *reinterpret_cast<const uint4 *>(A + m * K + c * 8);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  // A into TMEM columns [256, 256 + K/2): thread = row = lane of its warp quarter
  {
    uint32_t w[16];
    for (int blk = 0; blk < K / 32; ++blk) {
      for (int j = 0; j < 16; ++j) {
        const __nv_bfloat16 lo = A[row * K + blk * 32 + 2 * j], hi = A[row * K + blk * 32 + 2 * j + 1];
        w[j] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
      }
      tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + 256 + blk * 16, w);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16(128, N, 0);
    for (int k = 0; k < K / 16; ++k) {
      const uint64_t bd = sdesc_sw128(smem_u32(smem) + k * 32, 16, 1024);
      if (mode == 0) {
        umma_f16_ts(tmem, tmem + 256 + k * 8, bd, idesc, k != 0);
      } else {
        const uint64_t ad = sdesc_sw128(smem_u32(smem) + 16384 + k * 32, 16, 1024);
        umma_f16_ss(tmem, ad, bd, idesc, k != 0);
      }
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[row * N + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  __nv_bfloat16 hA[128 * K], hB[N * K];
  float fA[128 * K], fB[N * K];
  srand(1);
  for (int i = 0; i < 128 * K; ++i) { hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < N * K; ++i) { hB[i] = __float2bfloat16((rand() % 13 - 6) / 4.f); fB[i] = __bfloat162float(hB[i]); }
  __nv_bfloat16 *dA, *dB;
  float *dD, *hD = new float[128 * N];
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dD, 0, 128 * N * 4);
    k_ts<<<1, 128, 64 * 1024>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)fA[m * K + k] * fB[n * K + k];
        maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]));
      }
    printf("%s: max abs err %.3e (%s)\n", mode == 0 ? "TS (A in TMEM)" : "SS", maxerr, cudaGetErrorString(e));
  }
  return 0;
}
