// stack_bwd.cu -- backward of the TARGET side of the STCA stack, Eq.(3)-(9)
// (P:L112-156), trained end to end by Eq.(14).
//
// The history side of every layer (attention backward with the request-level aggregation of P:L396,
// then LN + SwiGLU-FFN backward of Eq.(2)) runs through the library's own kernels; the caller passes it
// in as `attn_hist` (one call per layer: dY -> dU, adding that layer's dX and history-weight
// gradients).  What is here is the part on the N_t target rows: small dense GEMMs (N_t x d x d..(M+1)d,
// cuBLAS SGEMM in fp32 -- plain library GEMMs, <1 % of the step's FLOPs) and row-wise kernels, in the
// reverse order of the forward:
//
//   forward recompute (fp32, from x_t and the forward's bf16 Y^(i) of every layer):
//     q1 = LN_Q1(SwiGLUFFN_Q1(x_t));  per layer cat_r = Y_r W_V^r, o = cat W_O,
//     c_(i+1) = [o1..oi | x_t] W_C(i+1), q_(i+1) = SwiGLUFFN_Q(i+1)(c_(i+1))
//   backward:
//     z:   dc_z = FFN_Z'(dz); dW_Z = [o1..oM | x_t]^T dc_z; d[o | x_t] += dc_z W_Z^T
//     layer i = M..1 (do_i complete):
//       dW_O = cat^T do_i; dcat = do_i W_O^T; dY_r = dcat_r W_V^r^T; dW_V^r = Y_r^T dcat_r
//       attn_hist(i): dY -> dU (dU = d loss / d U, U = q W_QK with W_QK^r = c W_Q^r W_K^r^T,
//                                c = log2(e) / sqrt(d_h))
//       qh = q_i W_Q; dqh_r = c dU_r W_K^r; dW_K^r = c dU_r^T qh_r; dW_Q = q_i^T dqh; dq = dqh W_Q^T
//       i >= 2: FFN_Q(i)' -> dc; dW_C(i) = [o1..o(i-1) | x_t]^T dc; d[o1..o(i-1) | x_t] += dc W_C(i)^T
//       i == 1: LN_Q1' and FFN_Q1' -> dx_t
#include <cublas_v2.h>
#include <math.h>

#include <algorithm>

#include "launch.h"

namespace stca {

namespace {

__global__ void k_swiglu32(const float *__restrict__ a, const float *__restrict__ g, float *__restrict__ H, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gv = g[i];
    H[i] = a[i] * (gv / (1.f + expf(-gv)));
  }
}

// da = dH silu(g), dg = dH a sig(g) (1 + g (1 - sig(g))), written over a and g
__global__ void k_swiglu_bwd32(float *__restrict__ a, float *__restrict__ g, const float *__restrict__ dH, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gv = g[i], av = a[i], sg = 1.f / (1.f + expf(-gv)), d = dH[i];
    a[i] = d * gv * sg;
    g[i] = d * av * sg * (1.f + gv * (1.f - sg));
  }
}

// one warp per row, PER = ceil(d / 32) values per lane (compile-time: small register arrays)
template <int PER>
__global__ void k_ln32(const float *__restrict__ y, const float *__restrict__ gam, const float *__restrict__ bet, int d,
                       int64_t rows, float eps, float *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    float v[PER], s1 = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k) v[k] = lane + 32 * k < d ? y[r * d + lane + 32 * k] : 0.f, s1 += v[k];
    const float mu = warp_sum(s1) / d;
    float s2 = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (lane + 32 * k < d) s2 += (v[k] - mu) * (v[k] - mu);
    const float inv = rsqrtf(warp_sum(s2) / d + eps);
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (lane + 32 * k < d) out[r * d + lane + 32 * k] = (v[k] - mu) * inv * gam[lane + 32 * k] + bet[lane + 32 * k];
  }
}

// LN backward, one warp per row, statistics recomputed from y; dy fp32; dgamma / dbeta per CTA in shared
// memory, then one atomic per column per CTA
template <int PER>
__global__ void __launch_bounds__(256) k_ln_bwd32(const float *__restrict__ y, const float *__restrict__ dout,
                                                  const float *__restrict__ gam, int d, int64_t rows, float eps,
                                                  float *__restrict__ dy, float *__restrict__ dgam, float *__restrict__ dbet) {
  extern __shared__ float acc[];  // [2][d]
  for (int e = threadIdx.x; e < 2 * d; e += blockDim.x) acc[e] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t r = (int64_t)blockIdx.x * 8 + w; r < rows; r += (int64_t)gridDim.x * 8) {
    float v[PER], gv[PER], s1 = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k) v[k] = lane + 32 * k < d ? y[r * d + lane + 32 * k] : 0.f, s1 += v[k];
    const float mu = warp_sum(s1) / d;
    float s2 = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (lane + 32 * k < d) s2 += (v[k] - mu) * (v[k] - mu);
    const float inv = rsqrtf(warp_sum(s2) / d + eps);
    float m1 = 0.f, m2 = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (lane + 32 * k < d) {
        const int e = lane + 32 * k;
        const float xh = (v[k] - mu) * inv, g = dout[r * d + e];
        atomicAdd(&acc[e], g * xh);
        atomicAdd(&acc[d + e], g);
        gv[k] = g * gam[e];
        v[k] = xh;
        m1 += gv[k];
        m2 += gv[k] * xh;
      }
    }
    m1 = warp_sum(m1) / d;
    m2 = warp_sum(m2) / d;
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (lane + 32 * k < d) dy[r * d + lane + 32 * k] = (gv[k] - m1 - v[k] * m2) * inv;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    atomicAdd(dgam + e, acc[e]);
    atomicAdd(dbet + e, acc[d + e]);
  }
}

// row-major C [m x n] = alpha op(A) [m x k] op(B) [k x n] + beta C, fp32 (cuBLAS is column-major: C^T = B^T A^T)
cublasStatus_t sg(cublasHandle_t hb, bool ta, bool tb, int m, int n, int k, float alpha, const float *A, int64_t lda,
                  const float *B, int64_t ldb, float beta, float *C, int64_t ldc) {
  return cublasSgemm(hb, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, n, m, k, &alpha, B, (int)ldb, A,
                     (int)lda, &beta, C, (int)ldc);
}

}  // namespace

size_t stack_bwd_scratch_bytes(int d, int h, int rd, int M, int64_t Nt) {
  const int64_t NQ = Nt * h;
  return (size_t)4 * ((size_t)Nt * d            // x_t fp32
                      + (size_t)M * Nt * d * 3     // q_i, c_i, cat_i
                      + (size_t)Nt * (M + 1) * d * 2  // [o1..oM | x_t] and its gradient
                      + (size_t)NQ * d * 3         // Y (fp32), dY, dU
                      + (size_t)Nt * rd * 4        // a, g, H, dH
                      + (size_t)Nt * d * 5) +      // yq1, dq, qh, dqh, t
         (size_t)64 * 256;
}

#define SG(...)                                                  \
  do {                                                           \
    if (sg(hb, __VA_ARGS__) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown; \
  } while (0)
#define CK(x)                          \
  do {                                 \
    cudaError_t e_ = (x);              \
    if (e_ != cudaSuccess) return e_;  \
  } while (0)

cudaError_t stack_bwd(void **blas, const StackBwd &a, cudaStream_t st) {
  if (!*blas) {
    cublasHandle_t hb;
    if (cublasCreate(&hb) != CUBLAS_STATUS_SUCCESS) return cudaErrorInitializationError;
    *blas = hb;
  }
  cublasHandle_t hb = (cublasHandle_t)*blas;
  if (cublasSetStream(hb, st) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  // the target side's fp32 GEMMs on the tensor cores in TF32 (10-bit mantissa products, fp32 accumulation:
  // finer than the bf16 operands the forward's target side uses); as SIMT SGEMMs they were ~10 % of the
  // training step (profiles/r2_final3_launches_stack_bwd.csv).  The history path's GEMMs (bf16 operands)
  // are not affected by the math mode.
  if (cublasSetMathMode(hb, CUBLAS_TF32_TENSOR_OP_MATH) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  const int d = a.d, h = a.h, rd = a.rd, M = a.M, dh = d / h;
  const int64_t Nt = a.Nt, NQ = Nt * h, ldo = (int64_t)(M + 1) * d;
  const int nt = (int)Nt;
  const float c = (float)(1.4426950408889634 / sqrt((double)dh));
  uint8_t *p = (uint8_t *)a.scratch;
  auto take = [&](size_t n) {
    float *q = (float *)p;
    p += (n * 4 + 255) / 256 * 256;
    return q;
  };
  float *xt = take((size_t)Nt * d);
  float *q[STCA_MAX_LAYERS], *cc[STCA_MAX_LAYERS], *cat[STCA_MAX_LAYERS];
  for (int i = 0; i < M; ++i) {
    q[i] = take((size_t)Nt * d);
    cc[i] = take((size_t)Nt * d);
    cat[i] = take((size_t)Nt * d);
  }
  float *oc = take((size_t)Nt * ldo), *dO = take((size_t)Nt * ldo);
  float *Y = take((size_t)NQ * d), *dY = take((size_t)NQ * d), *dU = take((size_t)NQ * d);
  float *A = take((size_t)Nt * rd), *G = take((size_t)Nt * rd), *H = take((size_t)Nt * rd), *dH = take((size_t)Nt * rd);
  float *yq1 = take((size_t)Nt * d), *dq = take((size_t)Nt * d), *qh = take((size_t)Nt * d), *dqh = take((size_t)Nt * d),
        *t = take((size_t)Nt * d);
  const int ew = 4 * sm_count();
  const int lnb = (int)std::min<int64_t>((Nt + 7) / 8, ew);
  auto ffn_fwd = [&](const float *x, const float *Wu, const float *Wv, const float *Wo, float *out) -> cudaError_t {
    SG(false, false, nt, rd, d, 1.f, x, d, Wu, rd, 0.f, A, rd);
    SG(false, false, nt, rd, d, 1.f, x, d, Wv, rd, 0.f, G, rd);
    note_launch();
    k_swiglu32<<<ew, 256, 0, st>>>(A, G, H, (int64_t)Nt * rd);
    SG(false, false, nt, d, rd, 1.f, H, rd, Wo, d, 0.f, out, d);
    return cudaGetLastError();
  };
  // dy -> dx (overwritten), dWu/dWv/dWo (accumulated); recomputes a, g, H from x
  auto ffn_bwd = [&](const float *x, const float *dy, const float *Wu, const float *Wv, const float *Wo, float *dx,
                     float *gWu, float *gWv, float *gWo) -> cudaError_t {
    SG(false, false, nt, rd, d, 1.f, x, d, Wu, rd, 0.f, A, rd);
    SG(false, false, nt, rd, d, 1.f, x, d, Wv, rd, 0.f, G, rd);
    note_launch();
    k_swiglu32<<<ew, 256, 0, st>>>(A, G, H, (int64_t)Nt * rd);
    SG(true, false, rd, d, nt, 1.f, H, rd, dy, d, 1.f, gWo, d);   // dWo += H^T dy
    SG(false, true, nt, rd, d, 1.f, dy, d, Wo, d, 0.f, dH, rd);   // dH = dy Wo^T
    note_launch();
    k_swiglu_bwd32<<<ew, 256, 0, st>>>(A, G, dH, (int64_t)Nt * rd);  // A = da, G = dg
    SG(true, false, d, rd, nt, 1.f, x, d, A, rd, 1.f, gWu, rd);   // dWu += x^T da
    SG(true, false, d, rd, nt, 1.f, x, d, G, rd, 1.f, gWv, rd);   // dWv += x^T dg
    SG(false, true, nt, d, rd, 1.f, A, rd, Wu, rd, 0.f, dx, d);   // dx = da Wu^T + dg Wv^T
    SG(false, true, nt, d, rd, 1.f, G, rd, Wv, rd, 1.f, dx, d);
    return cudaGetLastError();
  };

  // ---------------- forward recompute (fp32) ----------------
  CK(bf16_to_f32(a.xt, xt, Nt * d, st));
  CK(cudaMemcpy2DAsync(oc + (size_t)M * d, ldo * 4, xt, (size_t)d * 4, (size_t)d * 4, Nt, cudaMemcpyDeviceToDevice, st));
  CK(ffn_fwd(xt, a.qWu[0], a.qWv[0], a.qWo[0], yq1));
  note_launch();
  k_ln32<4><<<ew, 256, 0, st>>>(yq1, a.qg, a.qb, d, Nt, a.eps, q[0]);  // d = 128 (stca_backward's path)
  for (int i = 1; i <= M; ++i) {
    CK(bf16_to_f32(a.Y[i - 1], Y, NQ * d, st));
    for (int r = 0; r < h; ++r)  // cat_r = Y_r W_V[:, C_r]
      SG(false, false, nt, dh, d, 1.f, Y + (size_t)r * d, (int64_t)h * d, a.WV[i - 1] + r * dh, d, 0.f,
         cat[i - 1] + r * dh, d);
    SG(false, false, nt, d, d, 1.f, cat[i - 1], d, a.WO[i - 1], d, 0.f, oc + (size_t)(i - 1) * d, ldo);  // o_i
    if (i < M) {  // c_(i+1) = [o1..oi] W_C[0:i d] + x_t W_C[i d:(i+1) d]; q_(i+1) = FFN(c)
      SG(false, false, nt, d, i * d, 1.f, oc, ldo, a.WC[i], d, 0.f, cc[i], d);
      SG(false, false, nt, d, d, 1.f, xt, d, a.WC[i] + (size_t)i * d * d, d, 1.f, cc[i], d);
      CK(ffn_fwd(cc[i], a.qWu[i], a.qWv[i], a.qWo[i], q[i]));
    }
  }
  // ---------------- backward ----------------
  CK(cudaMemsetAsync(dO, 0, (size_t)Nt * ldo * 4, st));
  CK(cudaMemcpy2DAsync(dO, ldo * 4, a.dZ, (size_t)M * d * 4, (size_t)M * d * 4, Nt, cudaMemcpyDeviceToDevice, st));
  if (a.with_z && a.dz) {  // Eq.(9): input [o1..oM | x_t] is exactly oc
    SG(false, false, nt, d, (M + 1) * d, 1.f, oc, ldo, a.WZ, d, 0.f, t, d);  // c_z
    CK(ffn_bwd(t, a.dz, a.zWu, a.zWv, a.zWo, dq, a.g_zWu, a.g_zWv, a.g_zWo));
    SG(true, false, (M + 1) * d, d, nt, 1.f, oc, ldo, dq, d, 1.f, a.g_WZ, d);
    SG(false, true, nt, (M + 1) * d, d, 1.f, dq, d, a.WZ, d, 1.f, dO, ldo);
  }
  for (int i = M; i >= 1; --i) {
    const int L = i - 1;
    float *doi = dO + (size_t)L * d;
    CK(bf16_to_f32(a.Y[L], Y, NQ * d, st));
    SG(true, false, d, d, nt, 1.f, cat[L], d, doi, ldo, 1.f, a.g_WO[L], d);  // dW_O += cat^T do
    SG(false, true, nt, d, d, 1.f, doi, ldo, a.WO[L], d, 0.f, t, d);         // dcat
    for (int r = 0; r < h; ++r) {
      SG(false, true, nt, d, dh, 1.f, t + r * dh, d, a.WV[L] + r * dh, d, 0.f, dY + (size_t)r * d, (int64_t)h * d);
      SG(true, false, d, dh, nt, 1.f, Y + (size_t)r * d, (int64_t)h * d, t + r * dh, d, 1.f, a.g_WV[L] + r * dh, d);
    }
    CK(a.attn_hist(a.ctx, i, dY, dU));  // dY -> dU; history-side gradients of layer i
    SG(false, false, nt, d, d, 1.f, q[L], d, a.WQ[L], d, 0.f, qh, d);  // qh = q W_Q
    for (int r = 0; r < h; ++r) {
      SG(false, false, nt, dh, d, c, dU + (size_t)r * d, (int64_t)h * d, a.WK[L] + r * dh, d, 0.f, dqh + r * dh, d);
      SG(true, false, d, dh, nt, c, dU + (size_t)r * d, (int64_t)h * d, qh + r * dh, d, 1.f, a.g_WK[L] + r * dh, d);
    }
    SG(true, false, d, d, nt, 1.f, q[L], d, dqh, d, 1.f, a.g_WQ[L], d);  // dW_Q += q^T dqh
    SG(false, true, nt, d, d, 1.f, dqh, d, a.WQ[L], d, 0.f, dq, d);       // dq = dqh W_Q^T
    if (i >= 2) {  // Eq.(7): q_i = FFN_Q(i)(c_i), c_i = [o1..o(i-1) | x_t] W_C(i)
      CK(ffn_bwd(cc[L], dq, a.qWu[L], a.qWv[L], a.qWo[L], t, a.g_qWu[L], a.g_qWv[L], a.g_qWo[L]));
      SG(true, false, L * d, d, nt, 1.f, oc, ldo, t, d, 1.f, a.g_WC[L], d);
      SG(true, false, d, d, nt, 1.f, xt, d, t, d, 1.f, a.g_WC[L] + (size_t)L * d * d, d);
      SG(false, true, nt, L * d, d, 1.f, t, d, a.WC[L], d, 1.f, dO, ldo);
      SG(false, true, nt, d, d, 1.f, t, d, a.WC[L] + (size_t)L * d * d, d, 1.f, dO + (size_t)M * d, ldo);
    } else {  // Eq.(3): q1 = LN(FFN_Q1(x_t))
      note_launch();
      k_ln_bwd32<4><<<lnb, 256, 2 * d * sizeof(float), st>>>(yq1, dq, a.qg, d, Nt, a.eps, t, a.g_qg, a.g_qb);
      CK(ffn_bwd(xt, t, a.qWu[0], a.qWv[0], a.qWo[0], dq, a.g_qWu[0], a.g_qWv[0], a.g_qWo[0]));
      const float one = 1.f;
      if (cublasSgeam(hb, CUBLAS_OP_N, CUBLAS_OP_N, d, nt, &one, dO + (size_t)M * d, (int)ldo, &one, dq, d,
                      dO + (size_t)M * d, (int)ldo) != CUBLAS_STATUS_SUCCESS)
        return cudaErrorUnknown;
    }
  }
  if (a.dxt)
    CK(cudaMemcpy2DAsync(a.dxt, (size_t)d * 4, dO + (size_t)M * d, ldo * 4, (size_t)d * 4, Nt, cudaMemcpyDeviceToDevice, st));
  return cudaGetLastError();
}

}  // namespace stca
