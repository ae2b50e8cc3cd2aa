// tools/mma_bench.cu -- tcgen05.mma throughput microbenchmark (sm_100a), development aid.
// One CTA per SM, one thread issues `iters` MMAs back to back on fixed shared-memory
// operands; reports cycles per MMA instruction for several shapes / operand modes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2511_06077_b200/csrc mma_bench.cu -o mma_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace stca::tc;

template <int N, int BMN, int TS, int CE = 0>
__global__ void k_bench(int iters, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2[2];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2[0], 1);
    mbar_init(&bar2[1], 1);
    fence_mbar_init();
  }
  // zero operands
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = a + 32768;
    constexpr uint32_t idesc = idesc_bf16(128, N, BMN);
    // warm up
    for (int i = 0; i < 16; ++i) {
      const uint64_t ad = sdesc_sw128(a + (i & 3) * 32, 16, 1024);
      const uint64_t bd = BMN ? sdesc_sw128(b + (i & 3) * 2048, 16384, 1024) : sdesc_sw128(b + (i & 3) * 32, 16, 1024);
      if (TS) umma_f16_ts(tmem, tmem + 256, bd, idesc, 1); else umma_f16_ss(tmem, ad, bd, idesc, 1);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t ad = sdesc_sw128(a + (i & 3) * 32, 16, 1024);
      const uint64_t bd = BMN ? sdesc_sw128(b + (i & 3) * 2048, 16384, 1024) : sdesc_sw128(b + (i & 3) * 32, 16, 1024);
      if (TS) umma_f16_ts(tmem, tmem + 256, bd, idesc, 1); else umma_f16_ss(tmem, ad, bd, idesc, 1);
      if (CE && (i % CE) == CE - 1) umma_commit(&bar2[(i / CE) & 1]);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 1);
    const long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// the projection's per-chunk pattern: GEMM1 = 8 x (TS, N 128, B K-major) into G, then
// GEMM2 = 4 x (TS, N 128, B MN-major) into Y, with the kernel's commits (COMMITS = 0 / 1)
template <int C1, int C2>
__global__ void k_pattern(int iters, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bars[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t w1 = smem_u32(smem), wo = w1 + 65536;
    constexpr uint32_t id1 = idesc_bf16(128, 128, 0), id2 = idesc_bf16(128, 128, 1);
    long long t0 = 0;
    for (int it = -4; it < iters; ++it) {
      if (it == 0) {
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        t0 = clock64();
      }
      const int g = it & 1;
      for (int k = 0; k < 8; ++k)
        umma_f16_ts(tmem + 256 + g * 128, tmem + 128 + k * 8, sdesc_sw128(w1 + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024),
                    id1, k != 0);
      if (C1 >= 1) umma_commit(&bars[0]);
      if (C1 >= 2) umma_commit(&bars[1]);
      for (int k = 0; k < 4; ++k)
        umma_f16_ts(tmem, tmem + 192 + (g ^ 1) * 32 + k * 8, sdesc_sw128(wo + k * 2048, 8192, 1024), id2, 1);
      if (C2 >= 1) umma_commit(&bars[2]);
      if (C2 >= 2) umma_commit(&bars[3]);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 1);
    out[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int C1, int C2>
void run_pattern(const char *name) {
  unsigned long long *d, h;
  cudaMalloc(&d, 8);
  const int iters = 1024;
  cudaFuncSetAttribute(k_pattern<C1, C2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  k_pattern<C1, C2><<<1, 128, 96 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %7.1f cyc/chunk (ideal 768)  (%s)\n", name, (double)h / iters, cudaGetErrorString(e));
  cudaFree(d);
}

template <int N, int BMN, int TS, int CE = 0>
void run(const char *name, int grid) {
  unsigned long long *d, h[148];
  cudaMalloc(&d, sizeof h);
  const int iters = 4096;
  cudaFuncSetAttribute(k_bench<N, BMN, TS, CE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  k_bench<N, BMN, TS, CE><<<grid, 128, 96 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
  double cyc = (double)h[0] / iters;
  double macs = 128.0 * N * 16 / cyc;
  printf("%-32s grid %3d  %7.1f cyc/MMA  %7.0f MAC/cyc/SM  (%s)\n", name, grid, cyc, macs, cudaGetErrorString(e));
  cudaFree(d);
}

int main(int argc, char **argv) {
  if (argc > 1) {
    run_pattern<0, 0>("chunk 8 G1 + 4 G2: commits 0 / 0");
    run_pattern<1, 0>("chunk 8 G1 + 4 G2: commits 1 / 0");
    run_pattern<0, 1>("chunk 8 G1 + 4 G2: commits 0 / 1");
    run_pattern<1, 1>("chunk 8 G1 + 4 G2: commits 1 / 1");
    run_pattern<2, 1>("chunk 8 G1 + 4 G2: commits 2 / 1");
    run_pattern<2, 2>("chunk 8 G1 + 4 G2: commits 2 / 2");
    run<128, 0, 1>("TS M128 N128 B K-major", 1);
    run<128, 1, 1>("TS M128 N128 B MN-major", 1);
    run<128, 1, 0>("SS M128 N128 B MN-major", 1);
    return 0;
  }
  run<128, 0, 0, 1>("SS N128 commit every 1", 1);
  run<128, 0, 0, 4>("SS N128 commit every 4", 1);
  run<64, 0, 0, 8>("SS N64 commit every 8", 1);
  for (int grid : {1}) {
    run<64, 0, 0>("SS M128 N64  B K-major", grid);
    run<128, 0, 0>("SS M128 N128 B K-major", grid);
    run<256, 0, 0>("SS M128 N256 B K-major", grid);
    run<128, 1, 0>("SS M128 N128 B MN-major", grid);
    run<256, 1, 0>("SS M128 N256 B MN-major", grid);
    run<64, 0, 1>("TS M128 N64  B K-major", grid);
    run<128, 0, 1>("TS M128 N128 B K-major", grid);
    run<256, 0, 1>("TS M128 N256 B K-major", grid);
    run<128, 1, 1>("TS M128 N128 B MN-major", grid);
  }
  return 0;
}
