// tools/tmem_layout.cu -- which (TMEM lane, column) each thread / register of tcgen05.ld.16x256b and
// 16x32bx2 receives: TMEM is filled with value = lane * 1000 + column through 32x32b stores, then read
// back with the other shapes by warp 0 (lane base 0) and printed for a few threads.
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace stca::tc;

__global__ void k(float *out) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  {
    uint32_t w[32];
    for (int c0 = 0; c0 < 64; c0 += 32) {
      for (int j = 0; j < 32; ++j) w[j] = __float_as_uint((float)((warp * 32 + lane) * 1000 + c0 + j));
      tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + c0, w);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem));
    tmem_ld_wait();
    for (int i = 0; i < 8; ++i) out[lane * 8 + i] = __uint_as_float(r[i]);
    uint32_t q[4];
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], 8;"
                 : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3])
                 : "r"(tmem));
    tmem_ld_wait();
    for (int i = 0; i < 4; ++i) out[256 + lane * 4 + i] = __uint_as_float(q[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  float *d, h[384];
  cudaMalloc(&d, sizeof h);
  k<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("16x256b.x2 (%s): thread -> (lane*1000 + col) per register\n", cudaGetErrorString(e));
  for (int t = 0; t < 32; ++t) {
    printf("  t%2d:", t);
    for (int i = 0; i < 8; ++i) printf(" %6.0f", h[t * 8 + i]);
    printf("\n");
  }
  printf("16x32bx2.x4 imm 8:\n");
  for (int t = 0; t < 32; ++t) {
    printf("  t%2d:", t);
    for (int i = 0; i < 4; ++i) printf(" %6.0f", h[256 + t * 4 + i]);
    printf("\n");
  }
  return 0;
}
