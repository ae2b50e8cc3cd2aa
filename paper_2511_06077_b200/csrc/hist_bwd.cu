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
// The intermediates are bf16 (a and g come out of ONE GEMM with [Wu | Wv], rounded like the forward's
// operands), y stays fp32 for the LayerNorm statistics.  Rows are processed in blocks of 2^16 (working
// set ~0.5 GB at d = 128, r = 4).  Every history row
// appears once per request however many targets share it, so the gradients are aggregated at the
// request level by construction.
#include <cublas_v2.h>
#include <math.h>

#include <algorithm>

#include "launch.h"

namespace stca {

namespace {

__device__ __forceinline__ float silu_(float g) { return g / (1.f + __expf(-g)); }

// ag = [a | g] bf16 [n x 2rd] (a = X Wu, g = X Wv from one GEMM) -> h = a silu(g) bf16 [n x rd];
// 8 bf16 (16 bytes) per thread and access, rd % 8 == 0
__global__ void __launch_bounds__(256) k_swiglu_fwd(const bf16 *__restrict__ ag, bf16 *__restrict__ h, int rd, int64_t n) {
  const int per_row = rd / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * per_row; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / per_row;
    const int j = (int)(i - r * per_row);
    const uint4 av = *reinterpret_cast<const uint4 *>(ag + r * 2 * rd + 8 * j);
    const uint4 gv = *reinterpret_cast<const uint4 *>(ag + r * 2 * rd + rd + 8 * j);
    const __nv_bfloat162 *a2 = reinterpret_cast<const __nv_bfloat162 *>(&av), *g2 = reinterpret_cast<const __nv_bfloat162 *>(&gv);
    uint4 out;
    __nv_bfloat162 *o2 = reinterpret_cast<__nv_bfloat162 *>(&out);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 a = __bfloat1622float2(a2[k]), g = __bfloat1622float2(g2[k]);
      o2[k] = __floats2bfloat162_rn(a.x * silu_(g.x), a.y * silu_(g.y));
    }
    *reinterpret_cast<uint4 *>(h + r * rd + 8 * j) = out;
  }
}

// dag = [da | dg] bf16 [n x 2rd]: da = dH silu(g), dg = dH a sig(g) (1 + g (1 - sig(g)))
__global__ void __launch_bounds__(256) k_swiglu_bwd(const bf16 *__restrict__ ag, const bf16 *__restrict__ dh,
                                                    bf16 *__restrict__ dag, int rd, int64_t n) {
  const int per_row = rd / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * per_row; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / per_row;
    const int j = (int)(i - r * per_row);
    const uint4 av = *reinterpret_cast<const uint4 *>(ag + r * 2 * rd + 8 * j);
    const uint4 gv = *reinterpret_cast<const uint4 *>(ag + r * 2 * rd + rd + 8 * j);
    const uint4 dv = *reinterpret_cast<const uint4 *>(dh + r * rd + 8 * j);
    const __nv_bfloat162 *a2 = reinterpret_cast<const __nv_bfloat162 *>(&av), *g2 = reinterpret_cast<const __nv_bfloat162 *>(&gv),
                         *d2 = reinterpret_cast<const __nv_bfloat162 *>(&dv);
    uint4 oa, og;
    __nv_bfloat162 *oa2 = reinterpret_cast<__nv_bfloat162 *>(&oa), *og2 = reinterpret_cast<__nv_bfloat162 *>(&og);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 a = __bfloat1622float2(a2[k]), g = __bfloat1622float2(g2[k]), d = __bfloat1622float2(d2[k]);
      const float sx = 1.f / (1.f + __expf(-g.x)), sy = 1.f / (1.f + __expf(-g.y));
      oa2[k] = __floats2bfloat162_rn(d.x * g.x * sx, d.y * g.y * sy);
      og2[k] = __floats2bfloat162_rn(d.x * a.x * sx * (1.f + g.x * (1.f - sx)), d.y * a.y * sy * (1.f + g.y * (1.f - sy)));
    }
    *reinterpret_cast<uint4 *>(dag + r * 2 * rd + 8 * j) = oa;
    *reinterpret_cast<uint4 *>(dag + r * 2 * rd + rd + 8 * j) = og;
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

// Scratch is the caller's: ag, dag bf16 [R x 2rd]; h, dh bf16 [R x rd]; y fp32 [R x d]; dy bf16 [R x d]
size_t hist_bwd_scratch_bytes(int d, int rd, int64_t R) {
  return (size_t)R * rd * (4 * 2 + 2 * 2) + (size_t)R * d * (4 + 2) + 4096;
}

cudaError_t hist_bwd(void **blas, const bf16 *X, int64_t rows, int d, int rd, const bf16 *W1, const bf16 *Wo,
                     const float *gamma, float eps, const float *dXt, float *dX, float *dWu, float *dWv, float *dWo,
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
  bf16 *ag = (bf16 *)take((size_t)R * 2 * rd * 2), *dag = (bf16 *)take((size_t)R * 2 * rd * 2);
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
    // recompute the forward: [a | g] = X [Wu | Wv] (one GEMM, bf16), h = a silu(g) (bf16), y = h Wo (fp32)
    if (gemm_rm(hb, false, false, n, 2 * rd, d, Xb, d, W1, 2 * rd, ag, 2 * rd, 0.f, true) != CUBLAS_STATUS_SUCCESS)
      return cudaErrorUnknown;
    note_launch(3);
    k_swiglu_fwd<<<4 * ew, 256, 0, st>>>(ag, h, rd, (int64_t)n);
    if (gemm_rm(hb, false, false, n, d, rd, h, rd, Wo, d, y, d, 0.f) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
    // LayerNorm backward -> dy (bf16), dgamma, dbeta
    {
      const unsigned g = (unsigned)std::min<int64_t>((n + 7) / 8, 4 * ew);
      const size_t sm = 16 * d * sizeof(float);
      if (d <= 128) k_ln_bwd<4><<<g, 256, sm, st>>>(y, dXt + r0 * d, gamma, d, n, eps, dy, dgam, dbet);
      else if (d <= 256) k_ln_bwd<8><<<g, 256, sm, st>>>(y, dXt + r0 * d, gamma, d, n, eps, dy, dgam, dbet);
      else k_ln_bwd<16><<<g, 256, sm, st>>>(y, dXt + r0 * d, gamma, d, n, eps, dy, dgam, dbet);
    }
    // dWo += H^T dy;  dH = dy Wo^T (bf16)
    if (gemm_rm(hb, true, false, rd, d, n, h, rd, dy, d, dWo, d, 1.f) != CUBLAS_STATUS_SUCCESS ||
        gemm_rm(hb, false, true, n, rd, d, dy, d, Wo, d, dh, rd, 0.f, true) != CUBLAS_STATUS_SUCCESS)
      return cudaErrorUnknown;
    k_swiglu_bwd<<<4 * ew, 256, 0, st>>>(ag, dh, dag, rd, (int64_t)n);
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
