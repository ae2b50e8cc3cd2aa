// tools/tmem_bench.cu -- tcgen05.ld / tcgen05.st throughput by shape and warp count (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace stca::tc;

__device__ __forceinline__ void ld_16x256b_x8(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// MODE 0: 32x32b.x32 loads (thread = lane, 32 consecutive columns); MODE 1: 16x256b.x8 loads;
// MODE 2: 32x32b.x32 stores
template <int MODE>
__global__ void k_tmem(int iters, unsigned long long *out, uint32_t *sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t col0 = (warp >> 2) * 128;  // warps 4..7 use another column block
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 128; c += 32) {
      uint32_t r[32];
      if (MODE == 0) {
        tmem_ld32(tmem + lane_off + col0 + c, r);
      } else if (MODE == 1) {
        ld_16x256b_x8(tmem + lane_off + col0 + c, r);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = it + i;
        tmem_st32(tmem + lane_off + col0 + c, r);
      }
      if (MODE != 2) {
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) acc ^= r[i];
      }
    }
    if (MODE == 2) tmem_st_wait();
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
void run(const char *name, int warps) {
  unsigned long long *d, h;
  uint32_t *sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4096);
  const int iters = 256;
  k_tmem<MODE><<<1, 32 * warps>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  // bytes moved: per warp per iteration 32 lanes x 128 columns x 4 B (MODE 1: 16 lanes x ... same regs)
  const double bytes = (double)iters * warps * 32 * 128 * 4;
  printf("%-26s warps %d: %8.1f B/clk  (%s)\n", name, warps, bytes / (double)h, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int w : {4, 8}) {
    run<0>("ld 32x32b.x32", w);
    run<1>("ld 16x256b.x8", w);
    run<2>("st 32x32b.x32", w);
  }
  return 0;
}
