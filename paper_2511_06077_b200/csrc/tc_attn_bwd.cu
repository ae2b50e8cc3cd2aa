// tc_attn_bwd.cu -- backward of one layer's ragged single-query attention with request-level
// gradient aggregation (partial), d = 128, on tcgen05 (sm_100a).
//
// Forward (Eq.(13), the reordered form; U pre-scaled by log2(e)/sqrt(d_h)):
//   S = U_b X~_b^T,  alpha = 2^(S - m) / l,  Y = alpha X~_b.
// Backward, for dY = dLoss/dY:
//   D = rowsum(dY * Y) = rowsum(alpha * dP) with dP = dY X~_b^T
//   dS = ln2 alpha (dP - D),   dX~_b = alpha^T dY + dS^T U_b,   dU_b = dS X~_b.
// dX~_b sums over all of the request's query rows (m_b targets x h heads) INSIDE the MMA's K
// dimension: the history gradient is aggregated at the request level before it leaves the kernel
// ("aggregate gradients at the request level before synchronization").
//
// Transposed form (as tc_attn_narrow.cu): keys are the MMA's M (128 per tile), query rows its N
// (64 per work item).  Per key tile:
//   S^T, dP^T [128 x 64]  = X~_tile (K-major A) . U^T, dY^T (K-major B)            TMEM
//   dX~_tile  [128 x 128] = P^T (K-major A) . dY (MN-major B) + dS^T . U           TMEM -> global fp32
//   dU^T      [128 x 64] += X~_tile^T (MN-major A) . dS^T (MN-major B)             TMEM, across tiles
// Two passes over the item's keys: pass 1 takes each query row's exact maximum m, sum l and
// D = sum alpha dP (column reductions across the TMEM lanes: warp shuffles + 4 lane quarters through
// shared memory); pass 2 forms P = 2^(S - m) / l and dS, and runs the three gradient MMAs.  One CTA
// per work item (request, block of <= 64 query rows); a request with more query rows has several
// items, whose dX~ tiles are added with fp32 reductions (red.global.add) instead of stored.
#include <math.h>

#include "../../include/stca.h"
#include "launch.h"
#include "tc.h"
#include "tc_ptx.cuh"

namespace stca {
namespace tc {

bool make_map_bf16(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

struct BCfg {
  static constexpr int D = 128, BK = 128, NQ = 64;
  static constexpr int X_BYTES = BK * D * 2;     // 32 KB: two [128 keys x 64 d] SW128 boxes
  static constexpr int STAGES = 3;
  static constexpr int Q_BYTES = NQ * D * 2;     // 16 KB: U or dY block, two [64 x 64] boxes
  static constexpr int P_BYTES = BK * NQ * 2;    // 16 KB: P^T or dS^T, one [128 keys x 64 q] box
  static constexpr int RED_FLOATS = 2 * 4 * 32 * 2;  // [query half][lane quarter][32 columns] x 2 arrays
  static constexpr int SMEM = 1024 + STAGES * X_BYTES + 2 * Q_BYTES + 2 * P_BYTES + RED_FLOATS * 4 + 3 * 64 * 4 + 256;
  static constexpr uint32_t TS = 0, TP = 64, TX = 128, TU = 256;  // TMEM: S^T | dP^T | dX~ (128) | dU^T
  static constexpr int THREADS = 320;            // warps 0-7 compute, 8 TMA, 9 MMA
};

__host__ __device__ constexpr uint32_t idesc_bf16_amn_bmn(uint32_t M, uint32_t N) {
  return idesc_bf16(M, N, 1) | (1u << 15);
}

// v[c] (c < 32) over the warp's 32 lanes -> lane i returns op over all lanes of v[i]
template <bool MAX>
__device__ __forceinline__ float colreduce32(float (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = lane & s;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float keep = up ? v[i + s] : v[i], send = up ? v[i] : v[i + s];
      const float recv = __shfl_xor_sync(0xffffffffu, send, s);
      v[i] = MAX ? fmaxf(keep, recv) : keep + recv;
    }
  }
  return v[0];
}

__global__ void __launch_bounds__(BCfg::THREADS, 1)
    k_tc_attention_bwd(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapU,
                       const AttnItem *__restrict__ items, const float *__restrict__ dY, float *__restrict__ dX,
                       float *__restrict__ dU) {
  using C = BCfg;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *sX = smem;
  uint8_t *sU = sX + C::STAGES * C::X_BYTES;
  uint8_t *sDY = sU + C::Q_BYTES;
  uint8_t *sP = sDY + C::Q_BYTES;
  uint8_t *sDS = sP + C::P_BYTES;
  float *sRed = reinterpret_cast<float *>(sDS + C::P_BYTES);  // [2 arrays][2 qh][4 q][32]
  float *sM = sRed + C::RED_FLOATS, *sInvL = sM + 64, *sD = sInvL + 64;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sD + 64);
  uint64_t *x_full = bar, *x_empty = x_full + C::STAGES;
  uint64_t *u_full = x_empty + C::STAGES;  // TMA of U
  uint64_t *dy_ready = u_full + 1;         // 8 warps: dY block converted into SMEM
  uint64_t *s_full = dy_ready + 1, *s_free = s_full + 1;
  uint64_t *p_full = s_free + 1, *g_done = p_full + 1, *g_free = g_done + 1;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(g_free + 1);

  const AttnItem it = items[blockIdx.x];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nt = (it.klen + C::BK - 1) / C::BK;
  const bool accumulate = it.part_row != 0;  // several items share this request's keys: red.add dX~

  if (warp == 8 && lane == 0) {
    tma_prefetch(&mapX);
    tma_prefetch(&mapU);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&x_full[s], 1);
      mbar_init(&x_empty[s], 1);
    }
    mbar_init(u_full, 1);
    mbar_init(dy_ready, 8);
    mbar_init(s_full, 1);
    mbar_init(s_free, 8);
    mbar_init(p_full, 8);
    mbar_init(g_done, 1);
    mbar_init(g_free, 8);
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();

  if (warp == 8) {
    if (lane == 0) {  // ---------------- TMA: U, then the key tiles twice (pass 1, pass 2) ----------------
      mbar_expect_tx(u_full, C::Q_BYTES);
      tma_load_2d(sU, &mapU, u_full, 0, (int32_t)it.qrow0);
      tma_load_2d(sU + C::Q_BYTES / 2, &mapU, u_full, 64, (int32_t)it.qrow0);
      int s = 0, ph = 0;
      for (int g = 0; g < 2 * nt; ++g) {
        const int j = g < nt ? g : g - nt;
        mbar_wait(&x_empty[s], ph ^ 1);
        uint8_t *dst = sX + s * C::X_BYTES;
        const int32_t row = (int32_t)(it.key0 + (int64_t)j * C::BK);
        mbar_expect_tx(&x_full[s], C::X_BYTES);
        tma_load_2d(dst, &mapX, &x_full[s], 0, row);
        tma_load_2d(dst + C::X_BYTES / 2, &mapX, &x_full[s], 64, row);
        if (++s == C::STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      constexpr uint32_t id_s = idesc_bf16(128, C::NQ, 0);             // S^T, dP^T: B K-major
      constexpr uint32_t id_x = idesc_bf16(128, C::D, 1);              // dX~: A K-major, B MN-major
      constexpr uint32_t id_u = idesc_bf16_amn_bmn(128, C::NQ);        // dU^T: A, B MN-major
      const uint32_t aX = smem_u32(sX), aU = smem_u32(sU), aDY = smem_u32(sDY), aP = smem_u32(sP),
                     aDS = smem_u32(sDS);
      mbar_wait(u_full, 0);
      mbar_wait(dy_ready, 0);
      int s = 0, ph = 0;
      for (int g = 0; g < 2 * nt; ++g) {
        const int j = g < nt ? g : g - nt;
        mbar_wait(&x_full[s], ph);
        if (g >= 1) mbar_wait(s_free, (g - 1) & 1);  // S^T / dP^T of the previous tile loaded
        tc_fence_after();
        const uint32_t xs = aX + s * C::X_BYTES;
#pragma unroll
        for (int k = 0; k < C::D / 16; ++k) {
          const uint64_t ad = sdesc_sw128(xs + (k >> 2) * (C::X_BYTES / 2) + (k & 3) * 32, 16, 1024);
          umma_f16_ss(tmem + C::TS, ad, sdesc_sw128(aU + (k >> 2) * (C::Q_BYTES / 2) + (k & 3) * 32, 16, 1024), id_s,
                      k != 0);
          umma_f16_ss(tmem + C::TP, ad, sdesc_sw128(aDY + (k >> 2) * (C::Q_BYTES / 2) + (k & 3) * 32, 16, 1024),
                      id_s, k != 0);
        }
        umma_commit(s_full);
        if (g >= nt) {  // pass 2: the gradient MMAs of tile j
          mbar_wait(p_full, j & 1);
          if (j >= 1) mbar_wait(g_free, (j - 1) & 1);  // dX~ of tile j - 1 read out
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < C::NQ / 16; ++k) {  // dX~ = P^T dY + dS^T U (K = 64 query rows)
            umma_f16_ss(tmem + C::TX, sdesc_sw128(aP + k * 32, 16, 1024), sdesc_sw128(aDY + k * 2048, 8192, 1024), id_x,
                        k != 0);
          }
#pragma unroll
          for (int k = 0; k < C::NQ / 16; ++k)
            umma_f16_ss(tmem + C::TX, sdesc_sw128(aDS + k * 32, 16, 1024), sdesc_sw128(aU + k * 2048, 8192, 1024), id_x, 1);
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k)  // dU^T += X~^T dS^T (K = 128 keys)
            umma_f16_ss(tmem + C::TU, sdesc_sw128(xs + k * 2048, C::X_BYTES / 2, 1024),
                        sdesc_sw128(aDS + k * 2048, C::P_BYTES, 1024), id_u, (j | k) != 0);
          umma_commit(g_done);
        }
        umma_commit(&x_empty[s]);
        if (++s == C::STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {  // ---------------- compute warps: lane quarter q = keys 32q.., query half qh = columns 32qh.. ----------------
    const int q = warp & 3, qh = warp >> 2, tid = threadIdx.x;
    const uint32_t lanes = (uint32_t)(q * 32) << 16;
    const int key = q * 32 + lane;
    // dY block (fp32 global) -> bf16 in SMEM, the [64 x 128] layout of U (two SW128 boxes)
    for (int id = tid; id < C::NQ * 16; id += 256) {
      const int r = id >> 4, cc = id & 15;
      uint4 w = make_uint4(0, 0, 0, 0);
      if (r < it.nq) {
        const float4 *src = reinterpret_cast<const float4 *>(dY + (it.qrow0 + r) * C::D + cc * 8);
        const float4 a = src[0], b = src[1];
        w = make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
      }
      *reinterpret_cast<uint4 *>(sDY + (cc >> 3) * (C::Q_BYTES / 2) + sw128_off(r, cc & 7)) = w;
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(dy_ready);
    float mrun = -INFINITY, lrun = 0.f, drun = 0.f;  // lane i: statistics of query column 32 qh + i
    float *red0 = sRed + (qh * 4) * 32, *red1 = sRed + 2 * 4 * 32 + (qh * 4) * 32;
    for (int g = 0; g < 2 * nt; ++g) {
      const int j = g < nt ? g : g - nt;
      mbar_wait(s_full, g & 1);
      tc_fence_after();
      uint32_t sr[32], pr[32];
      tmem_ld32(tmem + lanes + C::TS + 32 * qh, sr);
      tmem_ld32(tmem + lanes + C::TP + 32 * qh, pr);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);
      const bool kv = key < it.klen - j * C::BK;
      if (g < nt) {  // ---- pass 1: exact column maximum, then sums of 2^(s-m) and 2^(s-m) dP ----
        float v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = kv ? __uint_as_float(sr[c]) : -INFINITY;
        const float wmax = colreduce32<true>(v, lane);
        red0[q * 32 + lane] = wmax;
        named_bar_sync(1 + qh, 128);
        float tmax = fmaxf(fmaxf(red0[lane], red0[32 + lane]), fmaxf(red0[64 + lane], red0[96 + lane]));
        const float mnew = fmaxf(mrun, tmax);
        float e[32], ed[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float mc = __shfl_sync(0xffffffffu, mnew, c);
          e[c] = kv ? ex2(__uint_as_float(sr[c]) - mc) : 0.f;
          ed[c] = e[c] * __uint_as_float(pr[c]);
        }
        const float se = colreduce32<false>(e, lane), sed = colreduce32<false>(ed, lane);
        named_bar_sync(1 + qh, 128);  // every warp of the half has read red0 / red1 of the last tile
        red0[q * 32 + lane] = se;
        red1[q * 32 + lane] = sed;
        named_bar_sync(1 + qh, 128);
        const float te = (red0[lane] + red0[32 + lane]) + (red0[64 + lane] + red0[96 + lane]);
        const float ted = (red1[lane] + red1[32 + lane]) + (red1[64 + lane] + red1[96 + lane]);
        const float f = mrun == -INFINITY ? 0.f : ex2(mrun - mnew);
        lrun = lrun * f + te;
        drun = drun * f + ted;
        mrun = mnew;
        named_bar_sync(1 + qh, 128);  // red0 / red1 reused by the next tile
        if (g == nt - 1) {  // the statistics of this half's 32 columns, for pass 2
          if (q == 0) {
            sM[32 * qh + lane] = mrun;
            sInvL[32 * qh + lane] = 1.f / lrun;
            sD[32 * qh + lane] = drun / lrun;
          }
          named_bar_sync(3, 256);
        }
      } else {  // ---- pass 2: P^T, dS^T -> SMEM; the previous tile's dX~ out ----
        uint32_t wp[16], wd[16];
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          float p2[2], d2[2];
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const int col = 32 * qh + c + e2;
            const bool ok = kv && col < it.nq;
            const float p = ok ? ex2(__uint_as_float(sr[c + e2]) - sM[col]) * sInvL[col] : 0.f;
            p2[e2] = p;
            d2[e2] = 0.69314718056f * p * (__uint_as_float(pr[c + e2]) - sD[col]);
          }
          wp[c / 2] = pack_bf16(p2[0], p2[1]);
          wd[c / 2] = pack_bf16(d2[0], d2[1]);
        }
        auto store_dx = [&](int jj) {  // dX~ tile jj: thread = key row, 64 of the d columns (half qh)
          mbar_wait(g_done, jj & 1);
          tc_fence_after();
          const bool kvj = key < it.klen - jj * C::BK;
          float *dst = dX + (it.key0 + (int64_t)jj * C::BK + key) * C::D + 64 * qh;
#pragma unroll 1
          for (int c = 0; c < 64; c += 32) {
            uint32_t o[32];
            tmem_ld32(tmem + lanes + C::TX + 64 * qh + c, o);
            tmem_ld_wait();
            if (kvj) {
              if (accumulate) {
#pragma unroll
                for (int e2 = 0; e2 < 32; ++e2) atomicAdd(dst + c + e2, __uint_as_float(o[e2]));
              } else {
#pragma unroll
                for (int e2 = 0; e2 < 32; e2 += 4)
                  *reinterpret_cast<float4 *>(dst + c + e2) =
                      make_float4(__uint_as_float(o[e2]), __uint_as_float(o[e2 + 1]), __uint_as_float(o[e2 + 2]),
                                  __uint_as_float(o[e2 + 3]));
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(g_free);
        };
        if (j >= 1) store_dx(j - 1);  // also: the MMAs of tile j - 1 are done with P^T / dS^T
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          *reinterpret_cast<uint4 *>(sP + sw128_off(key, 4 * qh + k)) = make_uint4(wp[4 * k], wp[4 * k + 1], wp[4 * k + 2], wp[4 * k + 3]);
          *reinterpret_cast<uint4 *>(sDS + sw128_off(key, 4 * qh + k)) = make_uint4(wd[4 * k], wd[4 * k + 1], wd[4 * k + 2], wd[4 * k + 3]);
        }
        fence_proxy_async();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        if (j == nt - 1) {
          store_dx(j);
          // dU^T (complete after the last tile): thread = d row (lane), 32 query columns of half qh
          uint32_t o[32];
          tmem_ld32(tmem + lanes + C::TU + 32 * qh, o);
          tmem_ld_wait();
#pragma unroll 4
          for (int c = 0; c < 32; ++c) {
            const int col = 32 * qh + c;
            if (col < it.nq) dU[(it.qrow0 + col) * C::D + key] = __uint_as_float(o[c]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc(tmem, 512);
}

}  // namespace tc

cudaError_t tc_attention_bwd(const void *U, int64_t NQ, const void *Xt, int64_t T2, const AttnItem *items,
                             int64_t n_items, const float *dY, float *dX, float *dU, cudaStream_t st) {
  using C = tc::BCfg;
  if (n_items <= 0) return cudaSuccess;
  CUtensorMap mx, mu;
  if (!tc::make_map_bf16(&mx, Xt, T2, C::D, C::D, C::BK) || !tc::make_map_bf16(&mu, U, NQ, C::D, C::D, C::NQ))
    return cudaErrorInvalidValue;
  cudaError_t e0 = smem_optin((const void *)tc::k_tc_attention_bwd, C::SMEM);
  if (e0 != cudaSuccess) return e0;
  note_launch();
  return launch_pdl(tc::k_tc_attention_bwd, dim3((unsigned)n_items), dim3(C::THREADS), (size_t)C::SMEM, st, mx, mu,
                    items, dY, dX, dU);
}

}  // namespace stca
