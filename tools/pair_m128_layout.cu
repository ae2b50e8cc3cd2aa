// tools/pair_m128_layout.cu -- where does a cta_group::2 M = 128 tcgen05.mma (kind::f16) put each
// CTA's 64 D rows in TMEM, can D start at TMEM lane 64 (or 16), and does the TS form (A from each
// CTA's TMEM) work with that layout?  A[128 x 16]: row i (CTA i / 64, local row i % 64) = i + 1 in
// column 0; B^T[64 x 16] column 0 = 1 (rows 0-31 in CTA 0, 32-63 in CTA 1), so D[i][n] = i + 1.
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2511_06077_b200/csrc tools/pair_m128_layout.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "tc_ptx.cuh"

using namespace stca::tc;
constexpr int N = 64;

__device__ __forceinline__ void umma_ts_pair(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// mode 0: SS, D lane base `base`; mode 1/2: TS with A in TMEM columns 256.. (layouts below), D at `base`
__global__ void __cluster_dims__(2, 1, 1) k(float *out, int base, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  if (warp == 0) tmem_alloc_pair(&tslot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 32 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (threadIdx.x < 64) {  // A: this CTA's 64 rows
    __nv_bfloat16 v = __float2bfloat16((float)(rank * 64 + threadIdx.x + 1));
    *reinterpret_cast<__nv_bfloat16 *>(smem + sw128_off(threadIdx.x, 0)) = v;
  }
  if (threadIdx.x < N / 2)  // B^T: this CTA's half of the N rows, B[n][0] = n + 1 (global n)
    *reinterpret_cast<__nv_bfloat16 *>(smem + 16384 + sw128_off(threadIdx.x, 0)) =
        __float2bfloat16((float)(rank * (N / 2) + threadIdx.x + 1));
  {
    uint32_t w[16];
    for (int i = 0; i < 16; ++i) w[i] = __float_as_uint(-1.f);
    for (int c = 0; c < N; c += 16) tmem_st16(tslot + ((uint32_t)(warp * 32) << 16) + c, w);
    // TS operand: lane l holds A row (l - base) of this CTA (for l in [base, base + 64)), packed bf16 pairs
    for (int i = 0; i < 16; ++i) w[i] = 0;
    const int l = warp * 32 + lane;
    // TS layouts tried: mode 1 = rows in lanes [base, base + 64), mode 2 = rows in lanes [64, 128) too (folded)
    if ((l >= base && l < base + 64) || (mode == 2 && l >= 64))
      w[0] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16((float)(rank * 64 + (l % 64) + 1)));
    tmem_st16(tslot + ((uint32_t)(warp * 32) << 16) + 256, w);
    tmem_st_wait();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t d = tmem + ((uint32_t)base << 16);
    if (mode == 0)
      umma_f16_ss_pair(d, sdesc_sw128(smem_u32(smem), 16, 1024), sdesc_sw128(smem_u32(smem) + 16384, 16, 1024),
                       idesc_bf16(128, N, 0), 0);
    else
      umma_ts_pair(d, tmem + ((uint32_t)base << 16) + 256, sdesc_sw128(smem_u32(smem) + 16384, 16, 1024),
                   idesc_bf16(128, N, 0), 0);
    umma_commit_pair_mc(&bar, 0x3);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[(rank * 128 + warp * 32 + lane) * N + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) tmem_dealloc_pair(tmem, 512);
}

int main(int argc, char **argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0, base = argc > 2 ? atoi(argv[2]) : 0;
  float *d, h[2 * 128 * N];
  cudaMalloc(&d, sizeof h);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  cudaMemset(d, 0, sizeof h);
  k<<<2, 128, 32 * 1024>>>(d, base, mode);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("mode %d (%s), D lane base %d (%s); D = (row + 1)(n + 1): per CTA and lane, the decoded (row, n) of columns 0, 1, 31\n",
         mode, mode ? "TS" : "SS", base, cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  for (int r = 0; r < 2; ++r)
    for (int l = 0; l < 128; l += (l % 32 == 0 || l % 32 == 31) ? 1 : 1) {
      const float *x = h + (r * 128 + l) * N;
      if (x[0] == -1.f && x[1] == -1.f) continue;
      printf("  %d.%3d:", r, l);
      for (int c : {0, 1, 31, 32, 63}) printf(" c%d=%g", c, x[c]);
      printf("\n");
    }
  return 0;
}
