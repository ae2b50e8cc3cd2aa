// kernels_cc.cu -- CUDA-core kernels: the fp32 path (STCA_FP32, 1e-4 parity) and
// utility kernels shared by both paths.  SURVEY §2.2 K-G; Eq.(1)-(9).
#include <math.h>

#include <stdio.h>
#include <stdlib.h>

#include "launch.h"

namespace stca {

// --------------------------------------------------------------------------
// tiled SGEMM-style GEMM, 64x64 tile, BK 16, 256 threads, 4x4 per thread
// --------------------------------------------------------------------------
template <typename S, int EPI>
__global__ void __launch_bounds__(256) k_cc_gemm(const S *__restrict__ A, int64_t lda, const S *__restrict__ B,
                                                 int64_t ldb, S *__restrict__ Cs, int64_t ldcs,
                                                 float *__restrict__ Cf, int64_t ldcf, int M, int N, int K,
                                                 float alpha) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      int r = i / 16, c = i % 16;  // A tile: 64 rows x 16 k
      int64_t gm = m0 + r;
      int gk = k0 + c;
      As[c][r] = (gm < M && gk < K) ? to_f(A[gm * lda + gk]) : 0.f;
      int rb = i / 64, cb = i % 64;  // B tile: 16 k x 64 cols
      int gkb = k0 + rb;
      int64_t gn = n0 + cb;
      Bs[rb][cb] = (gkb < K && gn < N) ? to_f(B[(int64_t)gkb * ldb + gn]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
    if (EPI == EPI_STORE) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int64_t gn = n0 + tx * 4 + j;
        if (gn >= N) continue;
        float v = alpha * acc[i][j];
        if (Cs) Cs[gm * ldcs + gn] = from_f<S>(v);
        if (Cf) Cf[gm * ldcf + gn] = v;
      }
    } else {  // SWIGLU: cols (2j, 2j+1) = (u_j, v_j) -> u * v * sigmoid(v), Eq.(1)
#pragma unroll
      for (int j = 0; j < 4; j += 2) {
        int64_t gn = n0 + tx * 4 + j;
        if (gn >= N) continue;
        float u = acc[i][j], v = acc[i][j + 1];
        float hv = u * (v / (1.f + expf(-v)));
        Cs[gm * ldcs + gn / 2] = from_f<S>(hv);
      }
    }
  }
}

cudaError_t cc_gemm(bool is_bf16, const void *A, int64_t lda, const void *B, int64_t ldb, void *Cs, int64_t ldcs,
                    float *Cf, int64_t ldcf, int M, int N, int K, float alpha, int epi, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  note_launch();
#define LAUNCH(S, E)                                                                                        \
  k_cc_gemm<S, E><<<grid, 256, 0, st>>>((const S *)A, lda, (const S *)B, ldb, (S *)Cs, ldcs, Cf, ldcf, M, N, \
                                        K, alpha)
  if (is_bf16) {
    if (epi == EPI_STORE) LAUNCH(bf16, EPI_STORE); else LAUNCH(bf16, EPI_SWIGLU);
  } else {
    if (epi == EPI_STORE) LAUNCH(float, EPI_STORE); else LAUNCH(float, EPI_SWIGLU);
  }
#undef LAUNCH
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// LayerNorm over rows, warp per row (biased variance, eps inside the sqrt)
// --------------------------------------------------------------------------
template <typename S>
__global__ void k_layernorm(const float *__restrict__ in, int64_t ldi, const float *__restrict__ g,
                            const float *__restrict__ b, float eps, S *__restrict__ out, int64_t ldo, int64_t rows,
                            int d) {
  int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x % 32;
  if (row >= rows) return;
  const float *x = in + row * ldi;
  float s = 0.f;
  for (int e = lane; e < d; e += 32) s += x[e];
  float mu = warp_sum(s) / d;
  float v = 0.f;
  for (int e = lane; e < d; e += 32) {
    float t = x[e] - mu;
    v += t * t;
  }
  float inv = rsqrtf(warp_sum(v) / d + eps);
  for (int e = lane; e < d; e += 32) out[row * ldo + e] = from_f<S>((x[e] - mu) * inv * g[e] + b[e]);
}

cudaError_t cc_layernorm(bool is_bf16, const float *in, int64_t ldi, const float *g, const float *b, float eps,
                         void *out, int64_t ldo, int64_t rows, int d, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  int64_t blocks = (rows + 7) / 8;
  note_launch();
  if (is_bf16)
    k_layernorm<bf16><<<(unsigned)blocks, 256, 0, st>>>(in, ldi, g, b, eps, (bf16 *)out, ldo, rows, d);
  else
    k_layernorm<float><<<(unsigned)blocks, 256, 0, st>>>(in, ldi, g, b, eps, (float *)out, ldo, rows, d);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// CUDA-core ragged single-query attention (reordered form, Eq.(13)).
// One CTA per work item: <= 16 query rows (2 per warp), keys streamed in tiles of 32
// through shared memory, online softmax in the log2 domain (U is pre-scaled by
// log2(e)/sqrt(d_h)).  Writes normalised Y rows (single-chunk requests) or
// (m, l, O) partials.
// --------------------------------------------------------------------------
// 16-byte (128-bit) loads of `n` storage elements at src -> fp32 in dst (n % (16 / sizeof(S)) == 0)
template <typename S>
__device__ __forceinline__ void unpack16(const uint4 v, float *dst) {
  if constexpr (sizeof(S) == 2) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      dst[2 * i] = __uint_as_float(w[i] << 16);
      dst[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  } else {
    dst[0] = __uint_as_float(v.x);
    dst[1] = __uint_as_float(v.y);
    dst[2] = __uint_as_float(v.z);
    dst[3] = __uint_as_float(v.w);
  }
}

// rows [r0, r0 + nr) of a row-major [* x d] storage matrix -> fp32 rows of stride dp in shared memory
// (zero past `valid` rows); 128-bit coalesced loads when a row is a whole number of 16-byte chunks
template <typename S>
__device__ __forceinline__ void load_rows_f32(const S *__restrict__ src, int64_t r0, int nr, int valid, int d, float *dst,
                                              int dp) {
  constexpr int V = 16 / sizeof(S);
  if (d % V == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int cpr = d / V;
    for (int i = threadIdx.x; i < nr * cpr; i += blockDim.x) {
      const int j = i / cpr, e = (i - j * cpr) * V;
      const uint4 v = j < valid ? __ldg(reinterpret_cast<const uint4 *>(src + (r0 + j) * d + e)) : make_uint4(0, 0, 0, 0);
      unpack16<S>(v, dst + j * dp + e);
    }
  } else {
    for (int i = threadIdx.x; i < nr * d; i += blockDim.x) {
      const int j = i / d, e = i % d;
      dst[j * dp + e] = j < valid ? to_f(src[(r0 + j) * d + e]) : 0.f;
    }
  }
}

template <typename S>
__global__ void __launch_bounds__(256) k_cc_attention(const S *__restrict__ U, const S *__restrict__ Xt,
                                                      const AttnItem *__restrict__ items, int d,
                                                      S *__restrict__ Y, float *__restrict__ part) {
  extern __shared__ float sm[];
  const AttnItem it = items[blockIdx.x];
  const int dp = d + 1;  // padded row (bank conflicts)
  float *Us = sm;             // [16][dp]
  float *Xs = Us + 16 * dp;   // [32][dp]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  load_rows_f32(U, it.qrow0, 16, it.nq, d, Us, dp);
  const int nd = (d + 31) / 32;  // dims per lane (<= 16)
  float O[2][16];
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
#pragma unroll
  for (int rr = 0; rr < 2; ++rr)
#pragma unroll
    for (int k = 0; k < 16; ++k) O[rr][k] = 0.f;
  for (int j0 = 0; j0 < it.klen; j0 += 32) {
    __syncthreads();
    const int nk = min(32, it.klen - j0);
    load_rows_f32(Xt, it.key0 + j0, 32, nk, d, Xs, dp);
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int q = warp * 2 + rr;
      if (q >= it.nq) continue;  // warp-uniform
      float s = 0.f;
      const float *ur = Us + q * dp, *xr = Xs + lane * dp;
      for (int e = 0; e < d; ++e) s = fmaf(ur[e], xr[e], s);
      if (lane >= nk) s = -INFINITY;
      float tmax = warp_max(s);
      float mnew = fmaxf(mrow[rr], tmax);
      float corr = exp2f(mrow[rr] - mnew);  // exp2(-inf) = 0 on the first tile
      float p = exp2f(s - mnew);
      lrow[rr] = lrow[rr] * corr + warp_sum(p);
      mrow[rr] = mnew;
#pragma unroll
      for (int k = 0; k < 16; ++k) O[rr][k] *= corr;
      for (int j = 0; j < nk; ++j) {
        float pj = __shfl_sync(0xffffffffu, p, j);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          int e = lane + 32 * k;
          if (k < nd && e < d) O[rr][k] = fmaf(pj, Xs[j * dp + e], O[rr][k]);
        }
      }
    }
  }
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int q = warp * 2 + rr;
    if (q >= it.nq) continue;
    if (it.part_row < 0) {
      const float inv = 1.f / lrow[rr];
      for (int k = 0; k < nd; ++k) {
        int e = lane + 32 * k;
        if (e < d) Y[(it.qrow0 + q) * d + e] = from_f<S>(O[rr][k] * inv);
      }
    } else {
      uint8_t *pr = reinterpret_cast<uint8_t *>(part) + (it.part_row + q) * (int64_t)part_row_bytes(d, sizeof(S));
      const float inv = 1.f / lrow[rr];
      if (lane == 0) *reinterpret_cast<float2 *>(pr + d * sizeof(S)) = make_float2(mrow[rr], lrow[rr]);
      for (int k = 0; k < nd; ++k) {
        int e = lane + 32 * k;
        if (e < d) reinterpret_cast<S *>(pr)[e] = from_f<S>(O[rr][k] * inv);
      }
    }
  }
}

cudaError_t cc_attention(bool is_bf16, const void *U, const void *Xt, const AttnItem *items, int64_t n_items, int d,
                         void *Y, float *part, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  size_t smem = sizeof(float) * (16 + 32) * (d + 1);
  note_launch();
  if (is_bf16) {
    cudaFuncSetAttribute(k_cc_attention<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_cc_attention<bf16><<<(unsigned)n_items, 256, smem, st>>>((const bf16 *)U, (const bf16 *)Xt, items, d,
                                                               (bf16 *)Y, part);
  } else {
    cudaFuncSetAttribute(k_cc_attention<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_cc_attention<float><<<(unsigned)n_items, 256, smem, st>>>((const float *)U, (const float *)Xt, items, d,
                                                                (float *)Y, part);
  }
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// split-K LSE merge (K-E): fold chunks 0..C-1 in order, per query row, from the normalised chunk
// outputs O^_c = O_c / l_c:  mu* = max_c mu_c;  w_c = 2^(mu_c - mu*) l_c;  Y = sum_c w_c O^_c / sum_c w_c
// (= sum_c 2^(mu_c - mu*) O_c / l*).  In split-history mode (G > 1) `part` holds every rank's
// partial buffer (rank-major, rank_stride BYTES) and chunk c of a request with C chunks is read from
// its owner rank floor(c G / C); with G = 1 this is the intra-GPU split-K merge.
// grid: (items, row blocks of 8 rows), warp per row.
// --------------------------------------------------------------------------
// PEER: the bytes live in another GPU's memory (written there by its own kernels), read through NVLink
// with L2-only loads (ld.global.cg) -- the SM's L1 is not coherent with a peer's writes, and a slot is
// reused every second layer
template <typename S, bool PEER>
__device__ __forceinline__ float4 load4(const uint8_t *p) {
  if constexpr (sizeof(S) == 4) {
    return PEER ? __ldcg(reinterpret_cast<const float4 *>(p)) : __ldg(reinterpret_cast<const float4 *>(p));
  } else {
    const uint2 v = PEER ? __ldcg(reinterpret_cast<const uint2 *>(p)) : __ldg(reinterpret_cast<const uint2 *>(p));
    return make_float4(__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u), __uint_as_float(v.y << 16),
                       __uint_as_float(v.y & 0xffff0000u));
  }
}

// split-history over peer memory: epoch flags between the ranks' kernels (no host, no collective
// library).  Rank g's flag words live in its own exchange buffer: ready[src] = the last epoch (layer
// of a forward) whose partials rank src has published.  A signal is one system-scope release store per
// peer after a system-scope fence; a wait spins on the rank's OWN memory with acquire loads.  A watchdog
// traps after 30 s without the peer (a peer that never arrives must not hang the GPU).
__device__ __forceinline__ void peer_signal_all(uint64_t *const *remote, int G, int me, uint64_t epoch) {
  __threadfence_system();
  for (int g = 0; g < G; ++g)
    if (g != me) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(remote[g] + me), "l"(epoch) : "memory");
}

__device__ __forceinline__ void peer_wait_all(const uint64_t *flags, int G, int me, uint64_t target) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int g = 0; g < G; ++g) {
    if (g == me) continue;
    for (;;) {
      uint64_t v, t;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + g) : "memory");
      if ((int64_t)v >= (int64_t)target) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 30000000000ull) {  // 30 s without the peer: fail loudly instead of hanging
        printf("stca peer wait: rank %d epoch %llu: rank %d is at %llu\n", me, (unsigned long long)target, g,
               (unsigned long long)v);
        __trap();
      }
      __nanosleep(32);
    }
  }
}

template <typename S, int MAXC, int RPW, bool PEER>
__global__ void __launch_bounds__(256) k_merge(const MergeItem *__restrict__ items, const uint8_t *__restrict__ part,
                                                const PeerMerge pm_, int d, int G, int64_t rank_stride,
                                                S *__restrict__ Y) {
  // MAXC: chunks per request handled in registers (C <= MAXC); RPW: rows per warp, all of their
  // loads issued before any use (the merge is latency-bound: more bytes in flight per thread)
  pdl_wait();  // the attention's partials are complete and visible
  pdl_trigger();
  const uint8_t *const *peer = pm_.slots;  // PEER: k_peer_exchange (the previous kernel) saw every peer's epoch
  const MergeItem it = items[blockIdx.x];
  const int lane = threadIdx.x % 32;
  const int qw = (blockIdx.y * 8 + threadIdx.x / 32) * RPW;  // this warp's first row
  if (qw >= it.rows) return;
  const int64_t rb = part_row_bytes(d, sizeof(S));
  const int64_t stride = (int64_t)it.rows * rb;
  const uint8_t *cb[MAXC];  // chunk c's partial lives in rank floor(c G / C)'s buffer (PEER: its own memory)
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    const int src = c < it.nchunks ? (c * G) / it.nchunks : 0;
    cb[c] = (PEER ? peer[src] : part + (int64_t)src * rank_stride) + (c < it.nchunks ? c * stride : 0);
  }
  const int e0 = lane * 4;
  float2 ml[RPW][MAXC];  // (m, l) of every row and chunk
  float4 a0[RPW][MAXC];  // and the first 128 output columns
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int64_t r0 = (it.part_row + qw + r) * rb;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      if (qw + r < it.rows && c < it.nchunks) {
        const float2 *pm = reinterpret_cast<const float2 *>(cb[c] + r0 + d * sizeof(S));
        ml[r][c] = PEER ? __ldcg(pm) : __ldg(pm);
        if (e0 < d) a0[r][c] = load4<S, PEER>(cb[c] + r0 + e0 * sizeof(S));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int q = qw + r;
    if (q >= it.rows) break;
    const int64_t r0 = (it.part_row + q) * rb;
    float mu = -INFINITY;
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c < it.nchunks) mu = fmaxf(mu, ml[r][c].x);
    float w[MAXC], l = 0.f;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      w[c] = 0.f;
      if (c < it.nchunks) {
        w[c] = exp2f(ml[r][c].x - mu) * ml[r][c].y;  // fold weight of chunk c (in chunk order below)
        l += w[c];
      }
    }
    const float inv = 1.f / l;
    for (int e = e0; e < d; e += 128) {  // d % 4 == 0: 4 elements per lane per step
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        if (c < it.nchunks) {
          const float4 a = e == e0 ? a0[r][c] : load4<S, PEER>(cb[c] + r0 + e * sizeof(S));
          acc.x += w[c] * a.x;
          acc.y += w[c] * a.y;
          acc.z += w[c] * a.z;
          acc.w += w[c] * a.w;
        }
      }
      S *yr = Y + (it.qrow0 + q) * d + e;
      if constexpr (sizeof(S) == 2) {  // four bf16 in one 8-byte store
        const __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
        const __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
        *reinterpret_cast<uint2 *>(yr) = make_uint2(*reinterpret_cast<const uint32_t *>(&lo),
                                                    *reinterpret_cast<const uint32_t *>(&hi));
      } else {
        *reinterpret_cast<float4 *>(yr) = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
      }
    }
  }
}

cudaError_t merge_partials(bool is_bf16, const MergeItem *items, int64_t n_items, int max_rows, int max_chunks,
                           const float *part, const PeerMerge *peer, int d, int G, int64_t rank_stride_bytes, void *Y,
                           cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  const uint8_t *p = (const uint8_t *)part;
  const PeerMerge pm = peer ? *peer : PeerMerge{};
  note_launch();
#define STCA_MERGE(S, MC, RPW)                                                                                      \
  do {                                                                                                             \
    const dim3 grid((unsigned)n_items, (unsigned)((max_rows + 8 * RPW - 1) / (8 * RPW)));                          \
    cudaError_t e = peer ? launch_pdl(k_merge<S, MC, RPW, true>, grid, dim3(256), 0, st, items, p, pm, d, G,        \
                                      rank_stride_bytes, (S *)Y)                                                   \
                         : launch_pdl(k_merge<S, MC, RPW, false>, grid, dim3(256), 0, st, items, p, pm, d, G,       \
                                      rank_stride_bytes, (S *)Y);                                                  \
    if (e != cudaSuccess) return e;                                                                                \
  } while (0)
  if (max_chunks <= 2) {  // the common case (a 10k history at the default cap): 4 rows per warp
    if (is_bf16) STCA_MERGE(bf16, 2, 4);
    else STCA_MERGE(float, 2, 4);
  } else {
    if (is_bf16) STCA_MERGE(bf16, 8, 1);
    else STCA_MERGE(float, 8, 1);
  }
#undef STCA_MERGE
  return cudaGetLastError();
}

// Fallback of the stream memory operations (api.cu peer_exchange_memops, STCA_PEER_KERNEL=1): publish
// this rank's epoch (its partials are complete: the attention kernel before it in the stream), then wait
// until every peer has published it; one thread of one CTA spins.
__global__ void k_peer_exchange(uint64_t *const *__restrict__ remote, const uint64_t *__restrict__ local, int G, int me,
                                uint64_t epoch) {
  pdl_wait();
  if (threadIdx.x == 0) {
    peer_signal_all(remote, G, me, epoch);
    peer_wait_all(local, G, me, epoch);
  }
}

cudaError_t peer_exchange(const PeerMerge &pm, int G, cudaStream_t st) {
  note_launch();
  k_peer_exchange<<<1, 32, 0, st>>>(pm.ready_remote, pm.ready_local, G, pm.me, pm.epoch);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------
// utilities
// --------------------------------------------------------------------------
__global__ void k_gather_rows(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst,
                              const int64_t *__restrict__ seg, int row_bytes) {
  const int64_t s = seg[blockIdx.y * 3 + 0], t = seg[blockIdx.y * 3 + 1], n = seg[blockIdx.y * 3 + 2];
  const int64_t bytes = n * row_bytes;
  const int64_t words = bytes / 16;  // row_bytes is a multiple of 16
  const int4 *s4 = reinterpret_cast<const int4 *>(src + s * row_bytes);
  int4 *t4 = reinterpret_cast<int4 *>(dst + t * row_bytes);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x)
    t4[i] = s4[i];
}

cudaError_t gather_rows(const void *src, void *dst, const int64_t *seg, int64_t nseg, int64_t max_len,
                        int row_bytes, cudaStream_t st) {
  if (nseg <= 0) return cudaSuccess;
  int64_t words = max_len * row_bytes / 16;
  unsigned gx = (unsigned)((words + 255) / 256);
  if (gx > 64) gx = 64;
  if (gx < 1) gx = 1;
  note_launch();
  k_gather_rows<<<dim3(gx, (unsigned)nseg), 256, 0, st>>>((const uint8_t *)src, (uint8_t *)dst, seg, row_bytes);
  return cudaGetLastError();
}

__global__ void k_copy_rows(const uint8_t *__restrict__ src, int64_t lds, uint8_t *__restrict__ dst, int64_t ldd,
                            int64_t rows, int row_bytes) {
  const int w = row_bytes / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * w; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / w, c = i % w;
    reinterpret_cast<uint32_t *>(dst + r * ldd)[c] = reinterpret_cast<const uint32_t *>(src + r * lds)[c];
  }
}

cudaError_t copy_rows_strided(const void *src, int64_t lds, void *dst, int64_t ldd, int64_t rows, int row_bytes,
                              cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  int64_t n = rows * (row_bytes / 4);
  unsigned g = (unsigned)((n + 255) / 256);
  if (g > 4096) g = 4096;
  note_launch();
  k_copy_rows<<<g, 256, 0, st>>>((const uint8_t *)src, lds, (uint8_t *)dst, ldd, rows, row_bytes);
  return cudaGetLastError();
}

// host-mapped pinned memory -> device, by SM loads over PCIe (no copy engine: a plan upload must not
// queue behind a large host-input copy in the H2D engine)
__global__ void k_fetch_mapped(const uint4 *__restrict__ src, uint4 *__restrict__ dst, int64_t n16) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

cudaError_t fetch_mapped(const void *src_mapped, void *dst, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  if ((bytes | (uintptr_t)src_mapped | (uintptr_t)dst) % 16) return cudaErrorInvalidValue;
  const int64_t n16 = (int64_t)(bytes / 16);
  unsigned g = (unsigned)((n16 + 255) / 256);
  if (g > 64) g = 64;
  note_launch();
  k_fetch_mapped<<<g, 256, 0, st>>>((const uint4 *)src_mapped, (uint4 *)dst, n16);
  return cudaGetLastError();
}

__global__ void k_f32_to_bf16(const float *__restrict__ s, bf16 *__restrict__ t, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    t[i] = __float2bfloat16_rn(s[i]);
}

cudaError_t f32_to_bf16(const float *src, bf16 *dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  unsigned g = (unsigned)((n + 255) / 256);
  if (g > 8192) g = 8192;
  note_launch();
  k_f32_to_bf16<<<g, 256, 0, st>>>(src, dst, n);
  return cudaGetLastError();
}

__global__ void k_bf16_to_f32(const bf16 *__restrict__ s, float *__restrict__ t, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    t[i] = __bfloat162float(s[i]);
}

cudaError_t bf16_to_f32(const bf16 *src, float *dst, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  unsigned g = (unsigned)((n + 255) / 256);
  if (g > 8192) g = 8192;
  note_launch();
  k_bf16_to_f32<<<g, 256, 0, st>>>(src, dst, n);
  return cudaGetLastError();
}

// W_QK^r = W_Q^r W_K^r^T (scaled) and W_VO^r = W_V^r W_O^r, one thread per output element.
__global__ void k_prep_qk_vo(const float *__restrict__ WQ, const float *__restrict__ WK,
                             const float *__restrict__ WV, const float *__restrict__ WO, int d, int h, float scale,
                             float *__restrict__ WQK, float *__restrict__ WVO) {
  const int dh = d / h;
  const int64_t total = (int64_t)h * d * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int r = (int)(i / ((int64_t)d * d));
    int e = (int)((i / d) % d), f = (int)(i % d);
    float qk = 0.f, vo = 0.f;
    for (int c = 0; c < dh; ++c) {
      qk = fmaf(WQ[(int64_t)e * d + r * dh + c], WK[(int64_t)f * d + r * dh + c], qk);
      vo = fmaf(WV[(int64_t)e * d + r * dh + c], WO[(int64_t)(r * dh + c) * d + f], vo);
    }
    WQK[(int64_t)e * (h * d) + (int64_t)r * d + f] = qk * scale;
    WVO[((int64_t)r * d + e) * d + f] = vo;
  }
}

cudaError_t prep_qk_vo(const float *WQ, const float *WK, const float *WV, const float *WO, int d, int h,
                       float qk_scale, float *WQK, float *WVO, cudaStream_t st) {
  int64_t total = (int64_t)h * d * d;
  unsigned g = (unsigned)((total + 255) / 256);
  if (g > 16384) g = 16384;
  note_launch();
  k_prep_qk_vo<<<g, 256, 0, st>>>(WQ, WK, WV, WO, d, h, qk_scale, WQK, WVO);
  return cudaGetLastError();
}

}  // namespace stca
