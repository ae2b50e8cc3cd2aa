// hist_bwd.cu -- backward of one layer's history path, Eq.(1)-(2), P:L103-111:
//   X~ = LN(SwiGLUFFN(X)) = LN((X Wu * silu(X Wv)) Wo) over the kept history rows.
//
// Per block of rows:
//   tc_ffn (tcgen05)        h = u silu(v) with [u | v] = X W1 (bf16, the SwiGLU epilogue: [u | v] stays on
//                           chip), y = h Wo (fp32) -- the forward recomputed, the LayerNorm's input
//   k_ln_bwd                per row: mu, s from y; x^ = (y - mu) / s; dx^ = dX~ * gamma;
//                           dy = (dx^ - mean(dx^) - x^ mean(dx^ x^)) / s -> bf16; dgamma += dX~ x^, dbeta += dX~
//   cuBLAS                  dWo += h^T dy;  dH = dy Wo^T (bf16)
//   tc_swiglu_bwd (tcgen05) [u | v] = X W1 recomputed in TMEM, the epilogue reads dH and writes
//                           da = dH silu(v), dv = dH u sig(v) (1 + v (1 - sig(v))) (bf16)
//   cuBLAS                  dWu += X^T da, dWv += X^T dv;  dX += [da | dv] [Wu | Wv]^T (one GEMM, K = 2 rd)
// (bf16 operands, fp32 accumulation.)  Rows are processed in blocks of 2^16.  Every history row
// appears once per request however many targets share it, so the gradients are aggregated at the
// request level by construction.
#include <cublas_v2.h>
#include <math.h>

#include <algorithm>

#include "launch.h"
#include "tc.h"

namespace stca {

namespace {

__device__ __forceinline__ uint32_t pack_bf16r(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&v);
}

// d = 128: a lane owns 4 consecutive columns (16-byte loads of y, dX~ and gamma, 8-byte stores of dy),
// a warp takes TWO rows per step with their shuffle reductions interleaved (the one-row, scalar-load
// form below ran at ~2.5 TB/s: latency-bound on its dependent warp sums)
__device__ __forceinline__ void warp_sum2(float &a, float &b) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
}
__global__ void __launch_bounds__(256) k_ln_bwd128(const float *__restrict__ y, const float *__restrict__ dXt,
                                                   const float *__restrict__ gamma, int64_t rows, float eps,
                                                   bf16 *__restrict__ dy, float *__restrict__ dgam,
                                                   float *__restrict__ dbet) {
  constexpr int D = 128;
  extern __shared__ float acc[];  // [8 warps][2][D]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float4 gm = reinterpret_cast<const float4 *>(gamma)[lane];
  float ga[4] = {0.f, 0.f, 0.f, 0.f}, ba[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t r0 = ((int64_t)blockIdx.x * 8 + w) * 2; r0 < rows; r0 += (int64_t)gridDim.x * 16) {
    float yv[2][4], dv[2][4];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const bool in = r0 + t < rows;
      const float4 a = in ? __ldg(reinterpret_cast<const float4 *>(y + (r0 + t) * D) + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 b = in ? __ldg(reinterpret_cast<const float4 *>(dXt + (r0 + t) * D) + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
      yv[t][0] = a.x; yv[t][1] = a.y; yv[t][2] = a.z; yv[t][3] = a.w;
      dv[t][0] = b.x; dv[t][1] = b.y; dv[t][2] = b.z; dv[t][3] = b.w;
    }
    float s0 = (yv[0][0] + yv[0][1]) + (yv[0][2] + yv[0][3]), s1 = (yv[1][0] + yv[1][1]) + (yv[1][2] + yv[1][3]);
    warp_sum2(s0, s1);
    const float mu[2] = {s0 / D, s1 / D};
    float q0 = 0.f, q1 = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      q0 += (yv[0][k] - mu[0]) * (yv[0][k] - mu[0]);
      q1 += (yv[1][k] - mu[1]) * (yv[1][k] - mu[1]);
    }
    warp_sum2(q0, q1);
    const float inv[2] = {rsqrtf(q0 / D + eps), rsqrtf(q1 / D + eps)};
    const float g4[4] = {gm.x, gm.y, gm.z, gm.w};
    float m1[2] = {0.f, 0.f}, m2[2] = {0.f, 0.f}, gv[2][4];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const bool in = r0 + t < rows;  // a missing second row has dv = 0: no gradient contribution
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float xh = (yv[t][k] - mu[t]) * inv[t], g = dv[t][k];
        if (in) {
          ga[k] += g * xh;
          ba[k] += g;
        }
        gv[t][k] = g * g4[k];
        yv[t][k] = xh;
        m1[t] += gv[t][k];
        m2[t] += gv[t][k] * xh;
      }
    }
    warp_sum2(m1[0], m1[1]);
    warp_sum2(m2[0], m2[1]);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (r0 + t >= rows) break;
      const float a = m1[t] / D, b = m2[t] / D;
      uint2 o;
      o.x = pack_bf16r((gv[t][0] - a - yv[t][0] * b) * inv[t], (gv[t][1] - a - yv[t][1] * b) * inv[t]);
      o.y = pack_bf16r((gv[t][2] - a - yv[t][2] * b) * inv[t], (gv[t][3] - a - yv[t][3] * b) * inv[t]);
      reinterpret_cast<uint2 *>(dy + (r0 + t) * D)[lane] = o;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    acc[(w * 2) * D + 4 * lane + k] = ga[k];
    acc[(w * 2 + 1) * D + 4 * lane + k] = ba[k];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < D; e += blockDim.x) {
    float sg = 0.f, sb = 0.f;
    for (int q = 0; q < 8; ++q) {
      sg += acc[(q * 2) * D + e];
      sb += acc[(q * 2 + 1) * D + e];
    }
    atomicAdd(dgam + e, sg);
    atomicAdd(dbet + e, sb);
  }
}

// one warp per row, PER = ceil(d / 32) values per lane (a template parameter: the register arrays stay
// small -- a runtime bound of 16 took 154 registers and 1/8 occupancy); a lane owns the same columns in
// every row, so dgamma / dbeta accumulate in its registers; the CTA's 8 warps combine in shared memory at
// the end, then one fp32 atomic per column per CTA
template <int PER>
__global__ void __launch_bounds__(256) k_ln_bwd(const float *__restrict__ y, const float *__restrict__ dXt,
                                                const float *__restrict__ gamma, int d, int64_t rows, float eps,
                                                bf16 *__restrict__ dy, float *__restrict__ dgam, float *__restrict__ dbet) {
  extern __shared__ float acc[];  // [8 warps][2][d]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float ga[PER], ba[PER], gm[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    ga[k] = ba[k] = 0.f;
    gm[k] = lane + 32 * k < d ? gamma[lane + 32 * k] : 0.f;
  }
  for (int64_t r = (int64_t)blockIdx.x * 8 + w; r < rows; r += (int64_t)gridDim.x * 8) {
    float yv[PER], gv[PER], dv[PER];
    float s1 = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k) {  // both rows' loads first (latency-bound kernel)
      const bool in = lane + 32 * k < d;
      yv[k] = in ? y[r * d + lane + 32 * k] : 0.f;
      dv[k] = in ? dXt[r * d + lane + 32 * k] : 0.f;
      s1 += yv[k];
    }
    const float mu = warp_sum(s1) / d;
    float s2 = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (lane + 32 * k < d) s2 += (yv[k] - mu) * (yv[k] - mu);
    const float inv = rsqrtf(warp_sum(s2) / d + eps);
    float m1 = 0.f, m2 = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const float xh = (yv[k] - mu) * inv, g = dv[k];
      ga[k] += g * xh;
      ba[k] += g;
      gv[k] = g * gm[k];
      yv[k] = xh;
      m1 += gv[k];
      m2 += gv[k] * xh;
    }
    m1 = warp_sum(m1) / d;
    m2 = warp_sum(m2) / d;
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (lane + 32 * k < d) dy[r * d + lane + 32 * k] = __float2bfloat16_rn((gv[k] - m1 - yv[k] * m2) * inv);
  }
#pragma unroll
  for (int k = 0; k < PER; ++k)
    if (lane + 32 * k < d) {
      acc[(w * 2) * d + lane + 32 * k] = ga[k];
      acc[(w * 2 + 1) * d + lane + 32 * k] = ba[k];
    }
  __syncthreads();
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    float sg = 0.f, sb = 0.f;
    for (int q = 0; q < 8; ++q) {
      sg += acc[(q * 2) * d + e];
      sb += acc[(q * 2 + 1) * d + e];
    }
    atomicAdd(dgam + e, sg);
    atomicAdd(dbet + e, sb);
  }
}

// row-major C [m x n] (+)= A [m x k] . B [k x n] with optional transposes, all row-major storage,
// bf16 operands, C in bf16 or fp32, fp32 compute (cuBLAS is column-major: C^T = B^T A^T)
cublasStatus_t gemm_rm(cublasHandle_t hb, bool ta, bool tb, int m, int n, int k, const void *A, int lda, const void *B,
                       int ldb, void *C, int ldc, float beta, bool c_bf16 = false) {
  const float alpha = 1.f;
  return cublasGemmEx(hb, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, n, m, k, &alpha, B,
                      CUDA_R_16BF, ldb, A, CUDA_R_16BF, lda, &beta, C, c_bf16 ? CUDA_R_16BF : CUDA_R_32F, ldc,
                      CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
}

}  // namespace

// Scratch is the caller's: dag bf16 [R x 2rd]; h, dh bf16 [R x rd]; y fp32 [R x d]; dy bf16 [R x d]
size_t hist_bwd_scratch_bytes(int d, int rd, int64_t R) {
  return (size_t)R * rd * (2 * 2 + 2 * 2) + (size_t)R * d * (4 + 2) + 4096;
}

cudaError_t hist_bwd(void **blas, const bf16 *X, int64_t rows, int d, int rd, const bf16 *W1, const bf16 *Wo,
                     const void *W1t, const void *Wot, const float *gamma, float eps, const float *dXt, float *dX, float *dWu, float *dWv, float *dWo,
                     float *dgam, float *dbet, void *scratch, int64_t R, cudaStream_t st) {
  if (!*blas) {
    cublasHandle_t hb;
    if (cublasCreate(&hb) != CUBLAS_STATUS_SUCCESS) return cudaErrorInitializationError;
    *blas = hb;
  }
  cublasHandle_t hb = (cublasHandle_t)*blas;
  if (cublasSetStream(hb, st) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  uint8_t *p = (uint8_t *)scratch;
  auto take = [&](size_t bytes) {
    void *q = p;
    p += (bytes + 255) / 256 * 256;
    return q;
  };
  bf16 *dag = (bf16 *)take((size_t)R * 2 * rd * 2);
  bf16 *h = (bf16 *)take((size_t)R * rd * 2), *dh = (bf16 *)take((size_t)R * rd * 2);
  float *y = (float *)take((size_t)R * d * 4);
  bf16 *dy = (bf16 *)take((size_t)R * d * 2);
  cudaError_t e;
  if ((e = cudaMemsetAsync(dWu, 0, (size_t)d * rd * 4, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(dWv, 0, (size_t)d * rd * 4, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(dWo, 0, (size_t)rd * d * 4, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(dgam, 0, (size_t)d * 4, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(dbet, 0, (size_t)d * 4, st)) != cudaSuccess) return e;
  const int ew = 4 * sm_count();
  for (int64_t r0 = 0; r0 < rows; r0 += R) {
    const int n = (int)std::min<int64_t>(R, rows - r0);
    const bf16 *Xb = X + r0 * d;
    // recompute the forward on tcgen05 (tc_ffn: the SwiGLU epilogue writes h = u silu(v) in bf16 and
    // [u | v] never reaches HBM; y = h Wo in fp32, the LayerNorm's input)
    if ((e = tc_ffn(Xb, d, n, W1t, Wot, d, rd, nullptr, nullptr, 0.f, nullptr, 0, y, d, h, st)) != cudaSuccess) return e;
    note_launch(1);
    // LayerNorm backward -> dy (bf16), dgamma, dbeta
    {
      const unsigned g = (unsigned)std::min<int64_t>((n + 7) / 8, 4 * ew);
      const size_t sm = 16 * d * sizeof(float);
      if (d == 128) k_ln_bwd128<<<(unsigned)std::min<int64_t>((n + 15) / 16, 4 * ew), 256, sm, st>>>(
          y, dXt + r0 * d, gamma, n, eps, dy, dgam, dbet);
      else if (d <= 128) k_ln_bwd<4><<<g, 256, sm, st>>>(y, dXt + r0 * d, gamma, d, n, eps, dy, dgam, dbet);
      else if (d <= 256) k_ln_bwd<8><<<g, 256, sm, st>>>(y, dXt + r0 * d, gamma, d, n, eps, dy, dgam, dbet);
      else k_ln_bwd<16><<<g, 256, sm, st>>>(y, dXt + r0 * d, gamma, d, n, eps, dy, dgam, dbet);
    }
    // dWo += H^T dy;  dH = dy Wo^T (bf16)
    if (gemm_rm(hb, true, false, rd, d, n, h, rd, dy, d, dWo, d, 1.f) != CUBLAS_STATUS_SUCCESS ||
        gemm_rm(hb, false, true, n, rd, d, dy, d, Wo, d, dh, rd, 0.f, true) != CUBLAS_STATUS_SUCCESS)
      return cudaErrorUnknown;
    // [da | dg] from the recomputed [u | v] = X W1 (tcgen05, in the GEMM's epilogue) and dH
    if ((e = tc_swiglu_bwd(Xb, d, n, W1t, d, rd, dh, rd, dag, 2 * rd, st)) != cudaSuccess) return e;
    // dWu += X^T da, dWv += X^T dg;  dX += [da | dg] [Wu | Wv]^T (one GEMM, K = 2 rd)
    float *dXb = dX + r0 * d;
    if (gemm_rm(hb, true, false, d, rd, n, Xb, d, dag, 2 * rd, dWu, rd, 1.f) != CUBLAS_STATUS_SUCCESS ||
        gemm_rm(hb, true, false, d, rd, n, Xb, d, dag + rd, 2 * rd, dWv, rd, 1.f) != CUBLAS_STATUS_SUCCESS ||
        gemm_rm(hb, false, true, n, d, 2 * rd, dag, 2 * rd, W1, 2 * rd, dXb, d, 1.f) != CUBLAS_STATUS_SUCCESS)
      return cudaErrorUnknown;
  }
  return cudaGetLastError();
}

void hist_bwd_release(void *blas) {
  if (blas) cublasDestroy((cublasHandle_t)blas);
}

}  // namespace stca
