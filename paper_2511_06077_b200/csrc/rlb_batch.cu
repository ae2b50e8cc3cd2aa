// rlb_batch.cu -- the training data path into the ragged forward:
// stochastic train lengths (Eq. beta-scale), temporal suffix, global length
// allocation against the budget B * L_avg (reading R-N2b) and sequence
// compaction with its segment map and ragged index.
//
// k_rlb_allocate: one CTA; B-sized integer work (reductions, O(B^2 / threads) ranking of the slack
//   pass, scan).  Exact: int64 and unsigned __int128 for req_b * budget; the only floating-point
//   decision (rounding L_raw to a multiple of 8) is taken in fp64 with explicit _rn ops, no FMA
//   contraction, in the oracle's operation order.
// k_rlb_gather: the HBM-bound copy of the kept suffix rows into the physical rows (read + write
//   of sum(alloc) * row_bytes); one warp per 4-KB range of P, 8 x 16-B streaming loads in flight per
//   lane, grid = 4 x 148 CTAs of 8 warps (all resident: <= 64 registers), plus one CTA that writes the segment map ((row, start,
//   len) triples per sequence) concurrently.
#include <stdint.h>

#include "launch.h"
#include "stca.h"

namespace {


constexpr int kAllocThreads = 1024;
constexpr int64_t kMaxB = 49152;   // 4 B of dynamic SMEM per sequence for the ranking

// exclusive block scan of one value per thread; returns the prefix, *total = block sum
__device__ int64_t block_exscan(int64_t v, int64_t *total) {
  __shared__ int64_t warp_sum[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sum[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t s = lane < (int)(blockDim.x >> 5) ? warp_sum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_sum[lane] = s;   // inclusive over warps
  }
  __syncthreads();
  const int64_t before = (w ? warp_sum[w - 1] : 0) + x - v;
  *total = warp_sum[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}

__global__ void __launch_bounds__(kAllocThreads) k_rlb_allocate(const double *__restrict__ s,
                                                                 const int64_t *__restrict__ hist_off, int64_t B,
                                                                 int32_t L_min, int32_t L_max, int64_t budget,
                                                                 int64_t *__restrict__ alloc,
                                                                 int64_t *__restrict__ new_off,
                                                                 int *__restrict__ status) {
  extern __shared__ int32_t trunc[];   // req_b - alloc_b if sequence b may take +8, else -1
  __shared__ int64_t s_total, s_slack;
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  // 1-2. L_train (Eq. beta-scale + rounding) and the temporal-suffix request; alloc <- req
  int64_t part = 0;
  for (int64_t b = threadIdx.x; b < B; b += blockDim.x) {
    const double sb = s[b];
    if (!(sb >= 0.0 && sb <= 1.0)) s_bad = 2;
    const double L_raw = __dadd_rn((double)L_min, __dmul_rn(sb, __dadd_rn((double)L_max, -(double)L_min)));
    const int64_t L_train = 8 * (int64_t)floor(__dadd_rn(L_raw / 8.0, 0.5));
    const int64_t n_b = hist_off[b + 1] - hist_off[b];
    const int64_t req = L_train < n_b ? L_train : n_b;
    alloc[b] = req;
    part += req;
  }
  {
    int64_t tot;
    block_exscan(part, &tot);
    if (threadIdx.x == 0) s_total = tot;
  }
  __syncthreads();
  const int64_t total = s_total;
  // 3. proportional scaling when over budget (exact), floor min(req, 8), one +8 per sequence
  if (total > budget) {
    part = 0;
    for (int64_t b = threadIdx.x; b < B; b += blockDim.x) {
      const int64_t req = alloc[b];
      const unsigned __int128 num = (unsigned __int128)req * (unsigned __int128)budget;
      int64_t a = 8 * (int64_t)(num / ((unsigned __int128)total * 8u));
      const int64_t fl = req < 8 ? req : 8;
      a = a > fl ? a : fl;
      trunc[b] = (a + 8 <= req) ? (int32_t)(req - a) : -1;
      alloc[b] = a;
      part += a;
    }
    int64_t sum;
    block_exscan(part, &sum);
    if (threadIdx.x == 0) {
      s_slack = budget - sum;
      if (s_slack < 0) s_bad = 1;
    }
    __syncthreads();
    const int64_t k = s_slack > 0 ? s_slack / 8 : 0;   // that many eligible sequences get +8
    if (k > 0) {
      for (int64_t b = threadIdx.x; b < B; b += blockDim.x) {
        const int32_t t = trunc[b];
        if (t < 0) continue;
        int64_t rank = 0;   // eligible sequences before b in (truncation desc, index asc)
        for (int64_t c = 0; c < B && rank < k; ++c) {
          const int32_t u = trunc[c];
          rank += (u > t) || (u == t && c < b);
        }
        if (rank < k) alloc[b] += 8;
      }
      __syncthreads();
    }
  }
  // ragged index over the compacted rows
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < B; b0 += blockDim.x) {
    const int64_t b = b0 + threadIdx.x;
    const int64_t v = b < B ? alloc[b] : 0;
    int64_t tot;
    const int64_t ex = block_exscan(v, &tot);
    if (b < B) new_off[b] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    new_off[B] = carry;
    *status = s_bad;  // 0 ok, 1 infeasible budget, 2 s outside [0, 1] (this call's own word)
  }
}

// the segment map, computed by one CTA (any multiple of 32 threads)
__device__ void rlb_segments(const int64_t *__restrict__ new_off, int64_t B, int32_t L_avg,
                             int64_t *__restrict__ seg_off, int64_t *__restrict__ segs) {
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < B; b0 += blockDim.x) {
    const int64_t b = b0 + threadIdx.x;
    int64_t p0 = 0, p1 = 0, cnt = 0;
    if (b < B) {
      p0 = new_off[b];
      p1 = new_off[b + 1];
      cnt = p1 > p0 ? (p1 - 1) / L_avg - p0 / L_avg + 1 : 0;
    }
    int64_t tot;
    const int64_t ex = carry + block_exscan(cnt, &tot);
    if (b < B) {
      seg_off[b] = ex;
      int64_t i = ex;
      for (int64_t p = p0; p < p1; ++i) {
        const int64_t row = p / L_avg, start = p - row * L_avg;
        const int64_t n = (p1 - p) < (L_avg - start) ? (p1 - p) : (L_avg - start);
        segs[3 * i + 0] = row;
        segs[3 * i + 1] = start;
        segs[3 * i + 2] = n;
        p += n;
      }
    }
    carry += tot;
  }
  if (threadIdx.x == 0) seg_off[B] = carry;
}

constexpr int kUnroll = 8;   // 16-B chunks in flight per lane
constexpr int kGatherThreads = 256;

// Each warp copies a contiguous range of 32 x kUnroll 16-B chunks of P (4 KB); lane l takes chunks
// l, l + 32, ...  A lane finds the sequence of its first chunk by binary search in new_off and walks
// forward for the rest (rows only increase), then issues all kUnroll loads before any store.
__global__ void __launch_bounds__(kGatherThreads, 4) k_rlb_gather(const uint4 *__restrict__ X,
                                                                const int64_t *__restrict__ hist_off,
                                                                const int64_t *__restrict__ alloc,
                                                                const int64_t *__restrict__ new_off, int64_t B,
                                                                int64_t cpr, int cpr_log2, int32_t L_avg,
                                                                int64_t *__restrict__ seg_off,
                                                                int64_t *__restrict__ segs, uint4 *__restrict__ P) {
  if (blockIdx.x == gridDim.x - 1) {   // the last CTA writes the segment map while the rest copy
    rlb_segments(new_off, B, L_avg, seg_off, segs);
    return;
  }
  const int64_t total = new_off[B] * cpr;   // chunks to write
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)(gridDim.x - 1) * (kGatherThreads / 32);
  constexpr int64_t kRange = 32 * kUnroll;
  for (int64_t c0 = ((int64_t)blockIdx.x * (kGatherThreads / 32) + (threadIdx.x >> 5)) * kRange; c0 < total;
       c0 += warps * kRange) {
    int64_t c = c0 + lane;
    if (c >= total) continue;
    int64_t p = cpr_log2 >= 0 ? c >> cpr_log2 : c / cpr;
    int64_t lo = 0, hi = B - 1;   // last b with new_off[b] <= p
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (__ldg(new_off + mid) <= p) lo = mid; else hi = mid - 1;
    }
    int64_t b = lo, nb = __ldg(new_off + b + 1), shift = (__ldg(hist_off + b + 1) - __ldg(alloc + b)) - __ldg(new_off + b);
    uint4 v[kUnroll];
    int64_t dst[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      c = c0 + lane + 32 * u;
      dst[u] = c < total ? c : -1;
      if (c < total) {
        p = cpr_log2 >= 0 ? c >> cpr_log2 : c / cpr;
        while (nb <= p) {   // next sequence (empty ones are skipped)
          ++b;
          nb = __ldg(new_off + b + 1);
          shift = (__ldg(hist_off + b + 1) - __ldg(alloc + b)) - __ldg(new_off + b);
        }
        v[u] = __ldcs(X + (p + shift) * cpr + (c - p * cpr));
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (dst[u] >= 0) __stcs(P + dst[u], v[u]);
  }
}

}  // namespace

extern "C" stca_status stca_rlb_allocate(const double *s, const int64_t *hist_off, int64_t B, int32_t L_min,
                                         int32_t L_max, int32_t L_avg, int64_t *alloc, int64_t *new_off,
                                         void *stream) {
  if (B < 1 || B > kMaxB || L_min < 0 || L_max < L_min || L_avg < 1 || !s || !hist_off || !alloc || !new_off)
    return STCA_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = (size_t)B * sizeof(int32_t);
  if (stca::smem_optin((const void *)k_rlb_allocate, (int)smem) != cudaSuccess) return STCA_ERR_CUDA;
  int *dstatus = nullptr;  // this call's status word (stream-ordered), never shared with another call
  if (cudaMallocAsync(&dstatus, sizeof(int), st) != cudaSuccess) {
    cudaGetLastError();
    return STCA_ERR_OOM;
  }
  k_rlb_allocate<<<1, kAllocThreads, smem, st>>>(s, hist_off, B, L_min, L_max, (int64_t)B * L_avg, alloc, new_off,
                                                 dstatus);
  stca::note_launch();
  const cudaError_t le = cudaGetLastError();
  int status = 0;
  const bool ok = le == cudaSuccess &&
                  cudaMemcpyAsync(&status, dstatus, sizeof(int), cudaMemcpyDeviceToHost, st) == cudaSuccess;
  cudaFreeAsync(dstatus, st);
  if (!ok || cudaStreamSynchronize(st) != cudaSuccess) {
    cudaGetLastError();
    return STCA_ERR_CUDA;
  }
  return status ? STCA_ERR_INVALID_ARG : STCA_OK;
}

extern "C" stca_status stca_rlb_compact(const void *X, int64_t row_bytes, const int64_t *hist_off,
                                        const int64_t *alloc, const int64_t *new_off, int64_t B, int32_t L_avg,
                                        void *P, int64_t *seg_off, int64_t *segs, void *stream) {
  if (B < 1 || L_avg < 1 || row_bytes < 16 || row_bytes % 16 || !X || !hist_off || !alloc || !new_off || !P ||
      !seg_off || !segs || ((uintptr_t)X | (uintptr_t)P) % 16)
    return STCA_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t cpr = row_bytes / 16;
  const int cpr_log2 = (cpr & (cpr - 1)) ? -1 : __builtin_ctzll((unsigned long long)cpr);
  k_rlb_gather<<<4 * stca::sm_count() + 1, kGatherThreads, 0, st>>>((const uint4 *)X, hist_off, alloc, new_off, B, cpr, cpr_log2,
                                                       L_avg, seg_off, segs, (uint4 *)P);
  stca::note_launch(1);
  return cudaGetLastError() == cudaSuccess ? STCA_OK : STCA_ERR_CUDA;
}
