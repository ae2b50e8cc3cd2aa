// encode.cu -- input-encoding prologue: the history rows X from ids.
//
// PAPER.md §3.1.1: x_j = video, action-type and position embeddings fused; time-delta side
// info: a per-token feature of request time minus item timestamp.  Fusion is additive
// (SPEC S:L130-138): x_j = E_v[v'_j] + E_a[a'_j] + E_p[p_j] (+ E_t[bucket_j]) with the readings of
// DESIGN.md R-N4a-c: p_j = recency rank (0 = most recent) clamped to the table, out-of-vocabulary ids
// to the tables' extra last row, bucket = floor(log2(dt)) for dt >= 1 (0 below), clamped.
//
// HBM-bound gather: one thread per 16-byte chunk of an output row (8 bf16 / 4 fp32), four 128-bit
// table loads in flight per thread, fp32 sum in the fixed order video + action + position + time,
// one 128-bit store; a resident grid (4 CTAs of 256 threads per SM) strides over T x chunks.  The
// request of a row is found by a binary search of hist_off (L1/L2-resident).  Algorithmic bytes per
// row: one video row (the large table; the others are L2-resident) + the output row + 24 B of ids.
#include <algorithm>

#include "../../include/stca.h"
#include "launch.h"

namespace {

__device__ __forceinline__ int64_t find_request(const int64_t *__restrict__ off, int64_t B, int64_t row) {
  int64_t lo = 0, hi = B;  // off[lo] <= row < off[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= row)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void add8(float (&acc)[8], uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    acc[2 * i] += __uint_as_float(w[i] << 16);
    acc[2 * i + 1] += __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

template <bool BF16>
__global__ void __launch_bounds__(256) k_encode(stca_embed_tables tab, int cpr /*16-B chunks per row*/,
                                                const int64_t *__restrict__ video_id,
                                                const int64_t *__restrict__ action_id,
                                                const int64_t *__restrict__ timestamp,
                                                const int64_t *__restrict__ hist_off, const int64_t *__restrict__ req_time,
                                                int64_t B, int64_t T, uint4 *__restrict__ X) {
  const uint4 *Ev = reinterpret_cast<const uint4 *>(tab.video), *Ea = reinterpret_cast<const uint4 *>(tab.action);
  const uint4 *Ep = reinterpret_cast<const uint4 *>(tab.position), *Et = reinterpret_cast<const uint4 *>(tab.tdelta);
  const int64_t n = T * cpr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / cpr;
    const int c = (int)(i - j * cpr);
    const int64_t b = find_request(hist_off, B, j);
    const int64_t last = __ldg(hist_off + b + 1) - 1;
    int64_t v = __ldg(video_id + j), a = __ldg(action_id + j);
    v = (v >= 0 && v < tab.n_video) ? v : tab.n_video;   // R-N4b: OOV row
    a = (a >= 0 && a < tab.n_action) ? a : tab.n_action;
    const int64_t p = min(last - j, tab.n_position - 1);  // R-N4a: recency rank
    const uint4 xv = __ldg(Ev + v * cpr + c), xa = __ldg(Ea + a * cpr + c), xp = __ldg(Ep + p * cpr + c);
    uint4 xt = make_uint4(0, 0, 0, 0);
    if (Et) {
      const int64_t dt = __ldg(req_time + b) - __ldg(timestamp + j);
      int64_t k = dt >= 1 ? 63 - __clzll((unsigned long long)dt) : 0;  // R-N4c: floor(log2(dt))
      k = min(k, tab.n_tdelta - 1);
      xt = __ldg(Et + k * cpr + c);
    }
    uint4 out;
    if (BF16) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      add8(acc, xv);
      add8(acc, xa);
      add8(acc, xp);
      if (Et) add8(acc, xt);
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
        w[q] = *reinterpret_cast<uint32_t *>(&h2);
      }
      out = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      const float4 fv = *reinterpret_cast<const float4 *>(&xv), fa = *reinterpret_cast<const float4 *>(&xa);
      const float4 fp = *reinterpret_cast<const float4 *>(&xp), ft = *reinterpret_cast<const float4 *>(&xt);
      float4 o = make_float4(fv.x + fa.x + fp.x, fv.y + fa.y + fp.y, fv.z + fa.z + fp.z, fv.w + fa.w + fp.w);
      if (Et) o = make_float4(o.x + ft.x, o.y + ft.y, o.z + ft.z, o.w + ft.w);
      out = *reinterpret_cast<uint4 *>(&o);
    }
    X[i] = out;
  }
}

}  // namespace

extern "C" stca_status stca_encode_history(const stca_embed_tables *tab, int32_t d, int32_t dtype,
                                           const int64_t *video_id, const int64_t *action_id,
                                           const int64_t *timestamp, const int64_t *hist_off,
                                           const int64_t *req_time, int64_t B, int64_t T, void *X, void *stream) {
  if (!tab || d <= 0 || B < 0 || T < 0 || (dtype != STCA_BF16 && dtype != STCA_FP32)) return STCA_ERR_INVALID_ARG;
  const int es = dtype == STCA_BF16 ? 2 : 4;
  if ((d * es) % 16) return STCA_ERR_UNSUPPORTED;
  if (T == 0) return STCA_OK;
  if (!X || !video_id || !action_id || !hist_off || !tab->video || !tab->action || !tab->position ||
      tab->n_video < 0 || tab->n_action < 0 || tab->n_position < 1 || (tab->tdelta && (tab->n_tdelta < 1 ||
      !timestamp || !req_time)) || ((uintptr_t)X | (uintptr_t)tab->video | (uintptr_t)tab->action |
      (uintptr_t)tab->position | (uintptr_t)tab->tdelta) % 16)
    return STCA_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int cpr = d * es / 16;
  const int64_t n = T * cpr;
  const int64_t grid = std::min<int64_t>((n + 255) / 256, 4 * (int64_t)stca::sm_count());
  stca::note_launch();
  if (es == 2)
    k_encode<true><<<(unsigned)grid, 256, 0, st>>>(*tab, cpr, video_id, action_id, timestamp, hist_off, req_time, B, T,
                                                   (uint4 *)X);
  else
    k_encode<false><<<(unsigned)grid, 256, 0, st>>>(*tab, cpr, video_id, action_id, timestamp, hist_off, req_time, B,
                                                    T, (uint4 *)X);
  return cudaGetLastError() == cudaSuccess ? STCA_OK : STCA_ERR_CUDA;
}
