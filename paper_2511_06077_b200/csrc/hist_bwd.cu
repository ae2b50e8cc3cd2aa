// hist_bwd.cu -- backward of one layer's history path (partial), Eq.(1)-(2),
// P:L103-111:  X~ = LN(SwiGLUFFN(X)) = LN((X Wu * silu(X Wv)) Wo) over the kept history rows.
//
// The plain GEMMs (recompute a = X Wu, g = X Wv, y = H Wo; then dH = dy Wo^T, dX = da Wu^T + dg Wv^T and
// the weight gradients dWo = H^T dy, dWu = X^T da, dWv = X^T dg, summed over all rows) are library GEMMs
// (cuBLAS, bf16 operands, fp32 accumulation); the two elementwise steps are kernels here:
//   k_swiglu_fwd   h = a * silu(g) -> bf16 (the forward's rounding point of H)
//   k_ln_bwd       per row: mu, s from y; x^ = (y - mu) / s; dx^ = dX~ * gamma;
//                  dy = (dx^ - mean(dx^) - x^ mean(dx^ x^)) / s -> bf16; dgamma += dX~ x^, dbeta += dX~
//   k_swiglu_bwd   da = dH silu(g), dg = dH a sig(g) (1 + g (1 - sig(g))) -> bf16
// Rows are processed in blocks of 2^16 (working set ~0.7 GB at d = 128, r = 4).  Every history row
// appears once per request however many targets share it, so the gradients are aggregated at the
// request level by construction.
#include <cublas_v2.h>
#include <math.h>

#include <algorithm>

#include "launch.h"

namespace stca {

namespace {

__global__ void k_swiglu_fwd(const float *__restrict__ a, const float *__restrict__ g, bf16 *__restrict__ h, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gv = g[i];
    h[i] = __float2bfloat16_rn(a[i] * (gv / (1.f + __expf(-gv))));
  }
}

__global__ void k_swiglu_bwd(const float *__restrict__ a, const float *__restrict__ g, const float *__restrict__ dh,
                             bf16 *__restrict__ da, bf16 *__restrict__ dg, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gv = g[i], sg = 1.f / (1.f + __expf(-gv)), d = dh[i];
    da[i] = __float2bfloat16_rn(d * gv * sg);
    dg[i] = __float2bfloat16_rn(d * a[i] * sg * (1.f + gv * (1.f - sg)));
  }
}

// one warp per row (d <= 512: 16 values per lane); dgamma / dbeta accumulated per CTA in shared
// memory, then one fp32 atomic per column per CTA
__global__ void __launch_bounds__(256) k_ln_bwd(const float *__restrict__ y, const float *__restrict__ dXt,
                                                const float *__restrict__ gamma, int d, int64_t rows, float eps,
                                                bf16 *__restrict__ dy, float *__restrict__ dgam, float *__restrict__ dbet) {
  extern __shared__ float acc[];  // [2][d]
  for (int e = threadIdx.x; e < 2 * d; e += blockDim.x) acc[e] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per = (d + 31) / 32;
  for (int64_t r = (int64_t)blockIdx.x * 8 + w; r < rows; r += (int64_t)gridDim.x * 8) {
    float yv[16], gv[16];
    float s1 = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < per && lane + 32 * k < d) s1 += (yv[k] = y[r * d + lane + 32 * k]);
    const float mu = warp_sum(s1) / d;
    float s2 = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < per && lane + 32 * k < d) s2 += (yv[k] - mu) * (yv[k] - mu);
    const float inv = rsqrtf(warp_sum(s2) / d + eps);
    float m1 = 0.f, m2 = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k < per && lane + 32 * k < d) {
        const int e = lane + 32 * k;
        const float xh = (yv[k] - mu) * inv, g = dXt[r * d + e];
        atomicAdd(&acc[e], g * xh);
        atomicAdd(&acc[d + e], g);
        gv[k] = g * gamma[e];
        yv[k] = xh;
        m1 += gv[k];
        m2 += gv[k] * xh;
      }
    }
    m1 = warp_sum(m1) / d;
    m2 = warp_sum(m2) / d;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < per && lane + 32 * k < d) dy[r * d + lane + 32 * k] = __float2bfloat16_rn((gv[k] - m1 - yv[k] * m2) * inv);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    atomicAdd(dgam + e, acc[e]);
    atomicAdd(dbet + e, acc[d + e]);
  }
}

// row-major C [m x n] (+)= A [m x k] . B [k x n] with optional transposes, all row-major storage,
// bf16 operands, fp32 C, fp32 compute (cuBLAS is column-major: C^T = B^T A^T)
cublasStatus_t gemm_rm(cublasHandle_t hb, bool ta, bool tb, int m, int n, int k, const void *A, int lda, const void *B,
                       int ldb, float *C, int ldc, float beta) {
  const float alpha = 1.f;
  return cublasGemmEx(hb, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, n, m, k, &alpha, B,
                      CUDA_R_16BF, ldb, A, CUDA_R_16BF, lda, &beta, C, CUDA_R_32F, ldc, CUBLAS_COMPUTE_32F,
                      CUBLAS_GEMM_DEFAULT);
}

}  // namespace

// Scratch is the caller's: a, g, dh fp32 [R x rd]; h, da, dg bf16 [R x rd]; y fp32 [R x d]; dy bf16 [R x d]
size_t hist_bwd_scratch_bytes(int d, int rd, int64_t R) {
  return (size_t)R * rd * (3 * 4 + 3 * 2) + (size_t)R * d * (4 + 2) + 4096;
}

cudaError_t hist_bwd(void **blas, const bf16 *X, int64_t rows, int d, int rd, const bf16 *Wu, const bf16 *Wv,
                     const bf16 *Wo, const float *gamma, float eps, const float *dXt, float *dX, float *dWu, float *dWv,
                     float *dWo, float *dgam, float *dbet, void *scratch, int64_t R, cudaStream_t st) {
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
  float *a = (float *)take((size_t)R * rd * 4), *g = (float *)take((size_t)R * rd * 4), *dh = (float *)take((size_t)R * rd * 4);
  bf16 *h = (bf16 *)take((size_t)R * rd * 2), *da = (bf16 *)take((size_t)R * rd * 2), *dg = (bf16 *)take((size_t)R * rd * 2);
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
    // recompute the forward: a = X Wu, g = X Wv, h = a silu(g) (bf16), y = h Wo
    if (gemm_rm(hb, false, false, n, rd, d, Xb, d, Wu, rd, a, rd, 0.f) != CUBLAS_STATUS_SUCCESS ||
        gemm_rm(hb, false, false, n, rd, d, Xb, d, Wv, rd, g, rd, 0.f) != CUBLAS_STATUS_SUCCESS)
      return cudaErrorUnknown;
    note_launch(3);
    k_swiglu_fwd<<<ew, 256, 0, st>>>(a, g, h, (int64_t)n * rd);
    if (gemm_rm(hb, false, false, n, d, rd, h, rd, Wo, d, y, d, 0.f) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
    // LayerNorm backward -> dy (bf16), dgamma, dbeta
    k_ln_bwd<<<std::min<int64_t>((n + 7) / 8, ew), 256, 2 * d * sizeof(float), st>>>(y, dXt + r0 * d, gamma, d, n, eps, dy,
                                                                                     dgam, dbet);
    // dWo += H^T dy;  dH = dy Wo^T
    if (gemm_rm(hb, true, false, rd, d, n, h, rd, dy, d, dWo, d, 1.f) != CUBLAS_STATUS_SUCCESS ||
        gemm_rm(hb, false, true, n, rd, d, dy, d, Wo, d, dh, rd, 0.f) != CUBLAS_STATUS_SUCCESS)
      return cudaErrorUnknown;
    k_swiglu_bwd<<<ew, 256, 0, st>>>(a, g, dh, da, dg, (int64_t)n * rd);
    // dWu += X^T da, dWv += X^T dg;  dX = da Wu^T + dg Wv^T
    float *dXb = dX + r0 * d;
    if (gemm_rm(hb, true, false, d, rd, n, Xb, d, da, rd, dWu, rd, 1.f) != CUBLAS_STATUS_SUCCESS ||
        gemm_rm(hb, true, false, d, rd, n, Xb, d, dg, rd, dWv, rd, 1.f) != CUBLAS_STATUS_SUCCESS ||
        gemm_rm(hb, false, true, n, d, rd, da, rd, Wu, rd, dXb, d, 1.f) != CUBLAS_STATUS_SUCCESS ||
        gemm_rm(hb, false, true, n, d, rd, dg, rd, Wv, rd, dXb, d, 1.f) != CUBLAS_STATUS_SUCCESS)
      return cudaErrorUnknown;
  }
  return cudaGetLastError();
}

void hist_bwd_release(void *blas) {
  if (blas) cublasDestroy((cublasHandle_t)blas);
}

}  // namespace stca
