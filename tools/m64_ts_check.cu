// tools/m64_ts_check.cu -- M = 64 TS MMA with the A operand in the UPPER lane half of TMEM
// (lane base 16: rows 0-15 -> lanes 16-31, 16-31 -> 48-63, ...) and D in the LOWER lane half
// (lane base 0), N = 256, K = 32; compared with a host reference.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "tc_ptx.cuh"

using namespace stca::tc;
constexpr int K = 32;
__constant__ int c_cfg[4];  // ts, a_lane, d_lane, n

__device__ __forceinline__ int row_of_lane(int lane128, int half) {  // M = 64 row held by a lane, or -1
  const int q = lane128 >> 5, l = lane128 & 31;
  if ((l >> 4) != half) return -1;
  return q * 16 + (l & 15);
}

template <int N>
__global__ void k(const __nv_bfloat16 *A /*[64 x K]*/, const __nv_bfloat16 *Bt /*[N x K]*/, float *D /*[64 x N]*/) {
  const int TS = c_cfg[0], AL = c_cfg[1], DL = c_cfg[2];
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, lane128 = threadIdx.x;
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int n = threadIdx.x; n < N; n += blockDim.x)
    for (int c = 0; c < K / 8; ++c)
      *reinterpret_cast<uint4 *>(smem + sw128_off(n, c)) = *reinterpret_cast<const uint4 *>(Bt + n * K + c * 8);
  for (int m = threadIdx.x; m < 64; m += blockDim.x)  // A for SS mode at smem + 32 KB
    for (int c = 0; c < K / 8; ++c)
      *reinterpret_cast<uint4 *>(smem + 32768 + sw128_off(m, c)) = *reinterpret_cast<const uint4 *>(A + m * K + c * 8);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  {  // A rows into the upper lane half, packed bf16 pairs, columns [320, 320 + K/2)
    const int r = row_of_lane(lane128, AL / 16);
    uint32_t w[16];
    for (int j = 0; j < 16; ++j) {
      uint32_t v = 0;
      if (r >= 0 && 2 * j + 1 < K)
        v = (uint32_t)__bfloat16_as_ushort(A[r * K + 2 * j]) | ((uint32_t)__bfloat16_as_ushort(A[r * K + 2 * j + 1]) << 16);
      w[j] = v;
    }
    tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + 320, w);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    for (int k = 0; k < K / 16; ++k)
      if (TS)
        umma_f16_ts(tmem + ((uint32_t)DL << 16), tmem + ((uint32_t)AL << 16) + 320 + k * 8,
                    sdesc_sw128(smem_u32(smem) + k * 32, 16, 1024), idesc_bf16(64, N, 0), k != 0);
      else
        umma_f16_ss(tmem + ((uint32_t)DL << 16), sdesc_sw128(smem_u32(smem) + 32768 + k * 32, 16, 1024),
                    sdesc_sw128(smem_u32(smem) + k * 32, 16, 1024), idesc_bf16(64, N, 0), k != 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int r = row_of_lane(lane128, DL / 16);
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    tmem_ld_wait();
    if (r >= 0)
      for (int j = 0; j < 16; ++j) D[r * N + c + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int N>
int runN(int ts, int al, int dl) {
  static __nv_bfloat16 hA[64 * K], hB[256 * K];
  static float fA[64 * K], fB[256 * K], hD[64 * 256];
  srand(3);
  for (int i = 0; i < 64 * K; ++i) { hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < N * K; ++i) { hB[i] = __float2bfloat16((rand() % 13 - 6) / 4.f); fB[i] = __bfloat162float(hB[i]); }
  __nv_bfloat16 *dA, *dB;
  float *dD;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, sizeof hD);
  int cfg[4] = {ts, al, dl, N};
  cudaMemcpyToSymbol(c_cfg, cfg, sizeof cfg);
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<N><<<1, 128, 64 * 1024>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, dD, 64 * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 64; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int kk = 0; kk < K; ++kk) ref += (double)fA[m * K + kk] * fB[n * K + kk];
      maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]));
    }
  printf("M64 %s A lane %d D lane %d N=%d: max abs err %.3e (%s)\n", ts ? "TS" : "SS", al, dl, N, maxerr,
         cudaGetErrorString(e));
  return 0;
}

int main(int argc, char **argv) {
  const int ts = atoi(argv[1]), al = atoi(argv[2]), dl = atoi(argv[3]), n = atoi(argv[4]);
  return n == 256 ? runN<256>(ts, al, dl) : runN<64>(ts, al, dl);
}
