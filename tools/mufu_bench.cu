// tools/mufu_bench.cu -- MUFU throughput on this GPU: ex2.approx / tanh.approx / rcp.approx (ops/clk/SM),
// and the FMA-pipe exp2 polynomial (ex2_fma) for comparison.
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

template <int OP>
__global__ void k(int iters, float *out, unsigned long long *cyc) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -(threadIdx.x + i) * 1e-3f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i]));
      if (OP == 1) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(a[i]));
      if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i]));
      if (OP == 3) y = stca::tc::ex2_fma(a[i]);
      if (OP == 4 || OP == 5) {  // packed half-precision tanh: two results per op (counted as 2)
        uint32_t x = __float_as_uint(a[i]), r;
        if (OP == 4) asm volatile("tanh.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x));
        else asm volatile("tanh.approx.bf16x2 %0, %1;" : "=r"(r) : "r"(x));
        y = __uint_as_float(r ^ 0x80008000u);
      }
      a[i] = y * -0.999f;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char *name) {
  float *o;
  unsigned long long *c, h;
  cudaMalloc(&o, 1 << 20);
  cudaMalloc(&c, 1024);
  const int iters = 2048, threads = 1024;
  k<OP><<<1, threads>>>(iters, o, c);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-22s %6.2f results/clk/SM\n", name, (double)iters * 8 * threads / h * (OP >= 4 ? 2 : 1));
}

int main() {
  run<0>("ex2.approx.ftz.f32");
  run<1>("tanh.approx.f32");
  run<2>("rcp.approx.ftz.f32");
  run<3>("ex2_fma (FMA pipe)");
  run<4>("tanh.approx.f16x2");
  run<5>("tanh.approx.bf16x2");
  return 0;
}
