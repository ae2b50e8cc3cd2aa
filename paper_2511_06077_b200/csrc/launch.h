// launch.h -- internal host-side launchers (C++ linkage, internal to libstca.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "common.cuh"
#include "stca.h"

namespace stca {

enum Epi { EPI_STORE = 0, EPI_SWIGLU = 1 };

// process-wide count of kernels launched by libstca (stca_kernel_launches())
void note_launch(int n = 1);

// Per-device launch setup (cudaFuncSetAttribute applies to the CURRENT device's context only, so a
// process-wide "done" flag would skip it for a handle on a second device).  Thread-safe, cached per
// (kernel, device ordinal).
cudaError_t smem_optin(const void *kernel, int bytes);   // MaxDynamicSharedMemorySize opt-in
int sm_count();                                          // SMs of the current device
// co-resident clusters of `cluster` CTAs of `kernel` (threads, smem) on the current device (>= 1)
int cluster_occupancy(const void *kernel, int threads, int smem, int cluster);

// Programmatic dependent launch for the forward's kernel chain: the kernel may be scheduled while
// its predecessor in the stream drains, so its launch and prologue (barrier init, TMEM alloc,
// tensor-map prefetch) overlap the predecessor's tail.  Every kernel launched this way executes
// griddepcontrol.wait (pdl_wait) before its first global-memory access, and signals its own
// dependents (pdl_trigger) right after its prologue.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- CUDA-core kernels (fp32 path; reference-grade, K-G of SURVEY §2.2) ----
// C = alpha * A[MxK] B[KxN]; A, B row-major storage S (lda, ldb);
// EPI_STORE: Cs (S, ldcs) and/or Cf (fp32, ldcf) get alpha*acc (either may be null);
// EPI_SWIGLU: B columns interleaved (u_j, v_j); Cs[:, j] = u_j * silu(v_j), N/2 output cols.
cudaError_t cc_gemm(bool is_bf16, const void *A, int64_t lda, const void *B, int64_t ldb, void *Cs, int64_t ldcs,
                    float *Cf, int64_t ldcf, int M, int N, int K, float alpha, int epi, cudaStream_t st);
// out (S, ldo) = LN(in fp32 [rows x d], ld) * g + b
cudaError_t cc_layernorm(bool is_bf16, const float *in, int64_t ldi, const float *g, const float *b, float eps,
                         void *out, int64_t ldo, int64_t rows, int d, cudaStream_t st);
// online-softmax sweep over items (qtile <= 16 rows per item)
cudaError_t cc_attention(bool is_bf16, const void *U, const void *Xt, const AttnItem *items, int64_t n_items, int d,
                         void *Y, float *part, cudaStream_t st);
// split-history over peer memory: peer_exchange publishes this rank's epoch and waits for every peer's
// (one spinning thread), then the merge reads chunk c from its owner's slot in place (kernels_cc.cu)
struct PeerMerge {
  const uint8_t *const *slots;   // device table: G ranks' partial slots of this epoch
  uint64_t *const *ready_remote; // device table: G ranks' ready-flag arrays
  const uint64_t *ready_local;   // this rank's ready flags (written by the peers)
  int me;
  uint64_t epoch;
};
// peer: NULL (part holds G rank-major copies when G > 1), or the peer-memory exchange of this layer
cudaError_t merge_partials(bool is_bf16, const MergeItem *items, int64_t n_items, int max_rows, int max_chunks,
                           const float *part, const PeerMerge *peer, int d, int G, int64_t rank_stride_bytes,
                           void *Y, cudaStream_t st);
cudaError_t peer_exchange(const PeerMerge &pm, int G, cudaStream_t st);

// ---- history-path backward (hist_bwd.cu; NEXT-1 partial) ----
size_t hist_bwd_scratch_bytes(int d, int rd, int64_t R);
// W1 = [Wu | Wv] bf16 [d x 2rd] (column blocks), Wo bf16 [rd x d]
cudaError_t hist_bwd(void **blas, const bf16 *X, int64_t rows, int d, int rd, const bf16 *W1, const bf16 *Wo,
                     const void *W1t, const void *Wot, const float *gamma, float eps, const float *dXt, float *dX, float *dWu, float *dWv, float *dWo,
                     float *dgam, float *dbet, void *scratch, int64_t R, cudaStream_t st);
void hist_bwd_release(void *blas);

// ---- target-side backward of the whole stack (stack_bwd.cu; NEXT-1) ----
// Weights fp32 in the user's [in x out] orientation; g_* gradients fp32, ACCUMULATED (zero them first).
// Per layer index L = i - 1; WC[0] / g_WC[0] unused.
struct StackBwd {
  int d, h, rd, M;
  float eps;
  bool with_z;
  int64_t Nt;
  const bf16 *xt;                        // [Nt x d]
  const bf16 *Y[STCA_MAX_LAYERS];        // the forward's attention outputs [Nt h x d]
  const float *dZ, *dz;                  // [Nt x M x d], [Nt x d] or NULL
  const float *qWu[STCA_MAX_LAYERS], *qWv[STCA_MAX_LAYERS], *qWo[STCA_MAX_LAYERS], *qg, *qb;
  const float *WQ[STCA_MAX_LAYERS], *WK[STCA_MAX_LAYERS], *WV[STCA_MAX_LAYERS], *WO[STCA_MAX_LAYERS];
  const float *WC[STCA_MAX_LAYERS], *WZ, *zWu, *zWv, *zWo;
  float *g_qWu[STCA_MAX_LAYERS], *g_qWv[STCA_MAX_LAYERS], *g_qWo[STCA_MAX_LAYERS], *g_qg, *g_qb;
  float *g_WQ[STCA_MAX_LAYERS], *g_WK[STCA_MAX_LAYERS], *g_WV[STCA_MAX_LAYERS], *g_WO[STCA_MAX_LAYERS];
  float *g_WC[STCA_MAX_LAYERS], *g_WZ, *g_zWu, *g_zWv, *g_zWo;
  float *dxt;                            // [Nt x d] written, or NULL
  // layer i's history side: dY [Nt h x d] -> dU [Nt h x d] (and that layer's dX / history-weight gradients)
  cudaError_t (*attn_hist)(void *ctx, int layer, const float *dY, float *dU);
  void *ctx;
  void *scratch;                         // stack_bwd_scratch_bytes
};
size_t stack_bwd_scratch_bytes(int d, int h, int rd, int M, int64_t Nt);
cudaError_t stack_bwd(void **blas, const StackBwd &a, cudaStream_t st);

// ---- utility kernels ----
cudaError_t gather_rows(const void *src, void *dst, const int64_t *seg /*[n][3]: src,dst,len*/, int64_t nseg,
                        int64_t max_len, int row_bytes, cudaStream_t st);
cudaError_t copy_rows_strided(const void *src, int64_t lds, void *dst, int64_t ldd, int64_t rows, int row_bytes,
                              cudaStream_t st);
cudaError_t f32_to_bf16(const float *src, bf16 *dst, int64_t n, cudaStream_t st);
// bytes (multiple of 16, 16-byte aligned) from host-mapped pinned memory to device memory by a kernel
cudaError_t fetch_mapped(const void *src_mapped, void *dst, size_t bytes, cudaStream_t st);
cudaError_t bf16_to_f32(const bf16 *src, float *dst, int64_t n, cudaStream_t st);
// WQK[e][r*d+f] = scale * sum_c WQ[e][r dh + c] WK[f][r dh + c];  WVO[r*d+e][f] = sum_c WV[e][r dh+c] WO[r dh+c][f]
cudaError_t prep_qk_vo(const float *WQ, const float *WK, const float *WV, const float *WO, int d, int h,
                       float qk_scale, float *WQK, float *WVO, cudaStream_t st);

}  // namespace stca
