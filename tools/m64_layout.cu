// tools/m64_layout.cu -- where does an M = 64 tcgen05.mma (cta_group::1, kind::f16) put its D rows
// in TMEM, and can D start at TMEM lane 64?  A[64 x 16] has row i = i+1 in column 0, B^T[N x 16]
// has column 0 = 1 for every n, so D[i][n] = i + 1 for all n: the dump shows each lane's row.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "tc_ptx.cuh"

using namespace stca::tc;
constexpr int N = 64;

__global__ void k(float *out, int lane_base) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  // A (K-major SW128, rows 0..63, 16 K): A[i][0] = i + 1
  if (threadIdx.x < 64) {
    __nv_bfloat16 v = __float2bfloat16((float)(threadIdx.x + 1));
    *reinterpret_cast<__nv_bfloat16 *>(smem + sw128_off(threadIdx.x, 0)) = v;
  }
  // B^T (K-major SW128, rows 0..N-1): B[n][0] = 1
  if (threadIdx.x < N) *reinterpret_cast<__nv_bfloat16 *>(smem + 16384 + sw128_off(threadIdx.x, 0)) = __float2bfloat16(1.f);
  // clear TMEM columns 0..N-1 of all lanes to -1
  {
    uint32_t w[16];
    for (int i = 0; i < 16; ++i) w[i] = __float_as_uint(-1.f);
    for (int c = 0; c < N; c += 16) tmem_st16(tslot + ((uint32_t)(warp * 32) << 16) + c, w);
    tmem_st_wait();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    umma_f16_ss(tmem + ((uint32_t)lane_base << 16), sdesc_sw128(smem_u32(smem), 16, 1024),
                sdesc_sw128(smem_u32(smem) + 16384, 16, 1024), idesc_bf16(64, N, 0), 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[(warp * 32 + lane) * N + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  float *d, h[128 * N];
  cudaMalloc(&d, sizeof h);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int base : {16, 32}) {
    k<<<1, 128, 64 * 1024>>>(d, base);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("D lane base %d (%s): lane -> value in columns 0 / 31 / 32 / 63\n", base, cudaGetErrorString(e));
    for (int l = 0; l < 128; ++l)
      printf("  lane %3d: %5.0f %5.0f %5.0f %5.0f%s", l, h[l * N], h[l * N + 31], h[l * N + 32], h[l * N + 63],
             (l % 2) ? "\n" : "");
  }
  return 0;
}
