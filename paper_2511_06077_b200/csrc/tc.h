// tc.h -- tcgen05 / TMEM / TMA kernels of the bf16 path (sm_100a), internal interface.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>

#include "common.cuh"

namespace stca {

// Repacked bf16 weights in K-major ("B^T", [N x K] row-major) layouts for TMA/UMMA.
struct TcWeights {
  void *W1h = nullptr;  // SwiGLU first GEMM, chunk-interleaved [u chunk | v chunk] rows, [2 rd x d]
  void *Woh = nullptr;  // W_o^T [d x rd]
  void *W1q = nullptr, *Woq = nullptr;  // query FFN of this layer (aliases W1h/Woh under reading R5)
  void *WQK = nullptr;  // W_QK^T [h d x d]
  void *WVO = nullptr;  // W_VO^T [d x h d]
  void *WC = nullptr;   // permuted W_C^T [d x i d] (or W_Z^T)
};

typedef std::function<void *(size_t)> DevAlloc;

struct TcProj {
  const void *X = nullptr;  // [rows x d] bf16
  int64_t rows = 0;
  int d = 0, rd = 0, M = 0;
  float eps = 1e-5f;
  const void *W1[16] = {}, *Wo[16] = {};
  const float *g[16] = {}, *b[16] = {};
  void *out = nullptr;            // layer i at out + i * out_layer_stride elements (bf16)
  int64_t out_layer_stride = 0;
  // two-GEMM path (d != 128): caller-owned H scratch of H_rows x rd bf16 (rows are processed in
  // pieces of at most H_rows)
  void *H = nullptr;
  int64_t H_rows = 0;
  // fused kernel (d == 128): all layers concatenated
  const void *W1cat = nullptr;    // [M x 2rd x d] bf16, per layer the chunk-interleaved W1^T
  const void *Wocat = nullptr;    // [M x rd x d] bf16, row-major W_o (MN-major B operand)
  const float *gcat = nullptr, *bcat = nullptr;  // [M x d]
};

struct TcProjWeights {
  void *W1cat = nullptr, *Wocat = nullptr;
  float *gcat = nullptr, *bcat = nullptr;
};
bool tc_prepare_proj(const float *const *Wu, const float *const *Wv, const float *const *Wo, const float *const *g,
                     const float *const *b, int M, int d, int rd, TcProjWeights *out, const DevAlloc &alloc);

bool tc_available();                       // sm_100a tensor-core path compiled in and usable
bool tc_attention_supported(int d);
bool tc_prepare_ffn(const float *Wu, const float *Wv, const float *Wo, int d, int rd, TcWeights *tc,
                    const DevAlloc &alloc);
// WQK/WVO: device bf16 row-major [d x hd] / [hd x d]; WC: device bf16 row-major [(i) d x d] (may be null)
bool tc_prepare_layer(const void *WQK, const void *WVO, const void *WC, int i, int d, int h, TcWeights *tc,
                      const DevAlloc &alloc);
cudaError_t tc_project(const TcProj &p, cudaStream_t st);
// SwiGLUFFN (+LN if g) over rows; outputs bf16 (out_s, ldo) and/or fp32 (out_f, ldof).  H: caller-owned
// scratch of at least rows * rd bf16 (the handle's, so concurrent handles / streams never share it)
cudaError_t tc_ffn(const void *in, int64_t ldi, int64_t rows, const void *W1, const void *Wo, int d, int rd,
                   const float *g, const float *b, float eps, void *out_s, int64_t ldo, float *out_f, int64_t ldof,
                   void *H, cudaStream_t st);
// SwiGLU gate backward on the recomputed [u | v] = X W1 (hist_bwd.cu): da -> dag[:, :rd], dv -> dag[:, rd:]
cudaError_t tc_swiglu_bwd(const void *X, int64_t ldx, int64_t rows, const void *W1, int d, int rd, const void *dH,
                          int64_t ldh, void *dag, int64_t lddag, cudaStream_t st);
// C[M x N] = A[M x K] (bf16, lda) . B where Bt = B^T [N x K] bf16 K-major
cudaError_t tc_gemm(const void *A, int64_t lda, const void *Bt, int64_t M, int N, int K, void *Cs, int64_t ldcs,
                    float *Cf, int64_t ldcf, cudaStream_t st);
// d in {256, 512}: 64-row query tiles, M = 64 MMAs, one-pass softmax with a lazy maximum (tc_attn_wide.cu)
// transposed ragged attention (keys as MMA rows) for requests with <= 64 query rows, d = 128
bool tc_attention_narrow_supported(int d, int max_rows);
// yh > 1: the standard form (Eq.(12)): U [N_t x yh d], keys [T2 x yh d], item.pad = head (api.cu);
// ncols = 64 or 32 query columns (every item of the launch has nq <= ncols)
cudaError_t tc_attention_narrow(const void *U, int64_t NQ, const void *Xt, int64_t T2, const AttnItem *items,
                                const int32_t *cta_off, const int32_t *cta_items, int n_ctas, void *Y, float *part,
                                cudaStream_t st, int yh, int ncols);
bool tc_attention_wide_supported(int d);
// The target-side update of one layer boundary as ONE kernel (d = 128; tc_chain.cu):
//   mode 0 (first): q(1) = LN(SwiGLUFFN(x_t)) -> U(1);  1 (mid): o(i) -> Z, ocat; c = ocat[:, :(i+1)d] W_C;
//   q = SwiGLUFFN(c) -> U(i+1);  2 (last): o(M) -> Z, ocat (and z = SwiGLUFFN_Z(ocat W_Z) if zout)
struct TcChain {
  int mode = 0, M = 0, h = 0, rd = 0;
  int64_t Nt = 0;
  int kc = 0;                      // K blocks of d of the c GEMM: i + 1 (mid), M + 1 (last with z)
  const void *Y = nullptr;         // [Nt x h d] bf16 (mid / last)
  const void *ocat = nullptr;      // [Nt x (M+1) d] bf16, read (x_t, earlier o)
  void *ocat_out = nullptr;        // ocat + i d: where o(i) goes
  float *Z = nullptr;              // out_Z + (i-1) d
  int64_t ldz = 0;
  void *U = nullptr;               // [Nt x h d] bf16 out (first / mid)
  float *zout = nullptr;           // [Nt x d] fp32 (last, with z)
  const void *WVOt = nullptr, *WCt = nullptr, *W1t = nullptr, *Wot = nullptr, *WQKt = nullptr;
  const float *g = nullptr, *b = nullptr;
  float eps = 1e-5f;
};
bool tc_chain_supported(int d, int h, int rd);
// NEXT-1 (partial): attention backward of one layer, d = 128; items of <= 64 query rows covering all of
// a request's keys (part_row != 0: dX~ accumulated with fp32 reductions, else stored)
cudaError_t tc_attention_bwd(const void *U, int64_t NQ, const void *Xt, int64_t T2, const AttnItem *items,
                             int64_t n_items, const float *dY, float *dX, float *dU, cudaStream_t st);
cudaError_t tc_chain(const TcChain &c, cudaStream_t st);
// d in {256, 512}: CTA pairs (cta_group::2, M = 128 = 64 query rows per CTA), items of <= 128 query rows
bool tc_attention_pair_supported(int d);
cudaError_t tc_attention_pair(const void *U, int64_t NQ, const void *Xt, int64_t T2, const AttnItem *items,
                              int64_t n_items, int d, void *Y, float *part, cudaStream_t st);
cudaError_t tc_attention_wide(const void *U, int64_t NQ, const void *Xt, int64_t T2, const AttnItem *items,
                              int64_t n_items, int d, void *Y, float *part, cudaStream_t st);
// d = 128, persistent: CTA c processes items[cta_items[cta_off[c] .. cta_off[c+1])] in order
int tc_attention_ctas();  // CTAs of the persistent attention grid (= SM count)
cudaError_t tc_attention(const void *U, int64_t NQ, const void *Xt, int64_t T2, const AttnItem *items,
                         const int32_t *cta_off, const int32_t *cta_items, int n_ctas, int d, void *Y, float *part,
                         cudaStream_t st);

}  // namespace stca
