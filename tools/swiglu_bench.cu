// tools/swiglu_bench.cu -- throughput of the projection's SwiGLU epilogue loop alone (no MMAs, no
// barriers): 8 warps in two groups, each group takes every other 128-row x 64-column chunk from TMEM
// (u | v, fp32), computes u * silu(v) in packed fp32x2 with tanh.approx, and stores bf16 H to TMEM.
// Reports cycles per chunk (the kernel's MMA time per chunk is 768).
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace stca::tc;

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t swiglu2(float u0, float v0, float u1, float v1) {
  const uint64_t v2 = f2_pack(v0, v1), half2 = f2_pack(0.5f, 0.5f);
  const uint64_t hv = f2_mul(v2, half2);
  const uint64_t t2 = f2_pack(tanh_approx(f2_lo(hv)), tanh_approx(f2_hi(hv)));
  const uint64_t sg = f2_fma(t2, half2, half2);
  const uint64_t uv = f2_mul(f2_pack(u0, u1), v2);
  const uint64_t h2 = f2_mul(uv, sg);
  return pack_bf16(f2_lo(h2), f2_hi(h2));
}

template <int MODE>  // 0: grouped (4 warps per chunk, 64 cols/thread); 1: all 8 warps per chunk (32 cols/thread)
__global__ void k(int nchunks, unsigned long long *out, uint32_t *sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int q = warp & 3, grp = warp >> 2;
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  {  // fill G buffers with something finite
    uint32_t w[32];
    for (int j = 0; j < 32; ++j) w[j] = __float_as_uint(0.01f * (j - 16 + lane));
    for (int c = 0; c < 256; c += 32) tmem_st32(tmem + lane_off + 256 + c, w);
    tmem_st_wait();
  }
  __syncthreads();
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int gc = 0; gc < nchunks; ++gc) {
    const int g = gc & 1;
    if (MODE == 0) {
      if (g != grp) continue;
      uint32_t h[32];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t u[32], v[32];
        tmem_ld32(tmem + lane_off + 256 + g * 128 + 32 * half, u);
        tmem_ld32(tmem + lane_off + 256 + g * 128 + 64 + 32 * half, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j)
          h[16 * half + j] = swiglu2(__uint_as_float(u[2 * j]), __uint_as_float(v[2 * j]), __uint_as_float(u[2 * j + 1]),
                                     __uint_as_float(v[2 * j + 1]));
      }
      tmem_st32(tmem + lane_off + 192 + g * 32, h);
      tmem_st_wait();
      acc ^= h[0];
    } else {
      uint32_t u[32], v[32], h[16];
      tmem_ld32(tmem + lane_off + 256 + g * 128 + 32 * grp, u);
      tmem_ld32(tmem + lane_off + 256 + g * 128 + 64 + 32 * grp, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j)
        h[j] = swiglu2(__uint_as_float(u[2 * j]), __uint_as_float(v[2 * j]), __uint_as_float(u[2 * j + 1]),
                       __uint_as_float(v[2 * j + 1]));
      tmem_st16(tmem + lane_off + 192 + g * 32 + 16 * grp, h);
      tmem_st_wait();
      acc ^= h[0];
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int MODE>
void run(const char *name, int extra_warps) {
  unsigned long long *d, h;
  uint32_t *sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4096);
  const int n = 512;
  k<MODE><<<1, 256 + 32 * extra_warps>>>(n, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %7.1f cycles/chunk (MUFU bound 512)  (%s)\n", name, (double)h / n, cudaGetErrorString(e));
}

int main() {
  run<0>("grouped: 4 warps/chunk, 64 cols/thread", 0);
  run<1>("8 warps/chunk, 32 cols/thread", 0);
  return 0;
}
