// tc_attn_narrow.cu -- ragged single-query attention for requests with few query rows
// (m_b * h <= 64, d = 128) on tcgen05, in the TRANSPOSED form.
//
// Same computation as tc_attn.cu (Eq.(13); Ragged Target Attention):
// per request, S = U_b X~_b^T, P = 2^(S - m), Y = P X~_b / sum, U pre-scaled by log2(e)/sqrt(d_h).
// With 8 targets x 4 heads = 32 query rows per request (the multi config) a 128-row query tile
// wastes 3/4 of every MMA and of the softmax, and the kernel stops being HBM-bound.  Here the keys
// are the MMA's M dimension and the queries its N dimension (N = NQ = 64, or 32 for requests with
// m_b h <= 32: a second instantiation chosen per request, P^T then in a SWIZZLE_64B layout):
//   S^T [128 keys x NQ queries]  = X~_tile (SMEM, K-major A) . U^T (SMEM, K-major B)
//   O^T [128 d    x NQ queries] += X~_tile^T (the SAME SMEM tile as an MN-major A) . P^T (SMEM, MN-major B)
// so the MMA work per key tile is 128 x NQ x 128 twice (not 128x128x128 twice) and a CTA streams X~ at
// HBM speed.  TMEM: S^T double buffer (2 x NQ columns) | O^T double buffer (2 x NQ columns).
//
// Softmax along TMEM lanes: a thread owns one key (lane) and NQ/4 query columns (four warps per
// lane quarter; with 8 warps of 32 columns the per-tile latency chain left the tile at ~2400 cycles).
// A query's running maximum is LAZY (as in tc_attn_wide.cu): a key tile only triggers the
// column-max reduction (recursive-halving shuffles per warp + 4 partials through SMEM) when
// some score exceeds the reference maximum by more than 2^8, which after the first tile is rare;
// then the affected O^T columns and sums are rescaled in place after the PVs so far completed.
// Sums stay per thread (per key, per query) until one reduction at the end of the item; at NQ = 32
// the item's output is written during the NEXT item's first tile (deferred epilogue, NCfg::DEFER).
//
// Warp roles (608 threads): 0..15 softmax (warp w: keys 32(w&3).., queries NQ/4 (w>>2)..) and output,
// 16 TMA producer, 17 TMEM allocator + S issuer, 18 PV issuer.  Persistent: one CTA per SM.
#include <math.h>

#include "launch.h"
#include "tc.h"
#include "tc_ptx.cuh"

#ifndef STCA_NARROW_LAZY
#define STCA_NARROW_LAZY 8.f  // rescale threshold in log2 units (a test build sets 0)
#endif
#ifndef STCA_NARROW_DEFER64
#define STCA_NARROW_DEFER64 0
#endif
#ifndef STCA_NARROW_FMA_NUM  // fraction of a thread's exponentials on the FMA pipe (A/B builds: 3 / 8 measured
#define STCA_NARROW_FMA_NUM 0  // 4 % slower at train and equal at multi -- MUFU does not bound this kernel,
#define STCA_NARROW_FMA_DEN 8  // profiles/r2_narrow_fma_ab)
#endif
#ifndef STCA_NARROW_PF
#define STCA_NARROW_PF 6  // key tiles prefetched into L2 ahead of the TMA loads (0: off)
#endif

namespace stca {
namespace tc {

bool make_map_bf16(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

template <int NQ_>
struct NCfg {
  static constexpr int D = 128, BK = 128, NQ = NQ_;   // d, keys per tile, query columns (64 or 32)
  static constexpr int CW = NQ / 4;                    // query columns per softmax warp (4 column groups)
  static constexpr int NFMA = STCA_NARROW_FMA_NUM * CW / STCA_NARROW_FMA_DEN;  // of them, exponentials on the FMA pipe
  static constexpr int X_BYTES = BK * D * 2;           // 2 boxes of 128 keys x 64 d (16 KB each)
  // 5 stages: a tile holds its slot from the TMA issue until its PV completes (~2 slots busy with
  // S / softmax / PV), so the slots left in flight bound the HBM bytes in flight per SM; the L2
  // prefetch (STCA_NARROW_PF tiles ahead) takes the HBM latency off the ring.  SMEM: 226.3 of 227 KB.
  static constexpr int STAGES = 5;
  static constexpr int P_BYTES = BK * NQ * 2;          // P^T: 128 keys x NQ queries, SW128 (NQ = 64) / SW64 (NQ = 32)
  static constexpr int U_BYTES = NQ * D * 2;           // U: 64 queries x 128 d, 2 boxes of 8 KB
  static constexpr int RED_BYTES = 4 * 4 * CW * 4;     // [column group][quarter][CW] column partials
  static constexpr int NSW = 16, THREADS = (NSW + 3) * 32;  // softmax warps; + producer, S / PV issuers
  // DEFERRED epilogue (an item's output written during the next item's first tile): at 32 columns;
  // at 64 the deferred item's state spills the tile loop (96 registers, measured slower: r2_narrow_defer)
  static constexpr bool DEFER = NQ == 32 || STCA_NARROW_DEFER64;
  // the deferred epilogue's copies of an item's column partial sums and reference maxima
  static constexpr int DEF_BYTES = DEFER ? RED_BYTES + 4 * CW * 4 : 0;
  static constexpr int USED = STAGES * X_BYTES + 2 * P_BYTES + 2 * U_BYTES + RED_BYTES + DEF_BYTES + 64 + 256;
  // 1 KB to align the base up to 1024 when it fits; at NQ = 64 it does not (227 KB), and the kernel
  // traps if the dynamic shared memory base is not 1024-aligned (it follows the 1 KB the system reserves)
  static constexpr int RESERVE = USED + 1024 <= 232448 ? 1024 : 0;
  static constexpr int SMEM = RESERVE + USED;
  static constexpr uint32_t TS = 0, TO = 128;          // S^T buffers at 0 / 64, O^T buffers at 128 / 192
};

// instruction descriptor with both operands MN-major (A = X~^T, B = P^T)
__host__ __device__ constexpr uint32_t idesc_bf16_mn(uint32_t M, uint32_t N) { return idesc_bf16(M, N, 1) | (1u << 15); }

// v[c], c < N (16 or 8), across the warp's 32 lanes -> lane i returns op over all lanes of v[i % N]
// (recursive halving over lane bits log2(N)-1..0, then butterflies over the remaining lane bits:
// 16 shuffles for N = 16, 9 for N = 8)
template <bool MAX, int N>
__device__ __forceinline__ float xreduce(float (&v)[N], int lane) {
#pragma unroll
  for (int s = N / 2; s >= 1; s >>= 1) {
    const bool up = lane & s;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float keep = up ? v[i + s] : v[i], send = up ? v[i] : v[i + s];
      const float recv = __shfl_xor_sync(0xffffffffu, send, s);
      v[i] = MAX ? fmaxf(keep, recv) : keep + recv;
    }
  }
  float r = v[0];
#pragma unroll
  for (int s = N; s < 32; s <<= 1) {
    const float o = __shfl_xor_sync(0xffffffffu, r, s);
    r = MAX ? fmaxf(r, o) : r + o;
  }
  return r;
}

template <int N>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 16) tmem_ld16(taddr, r);
  else tmem_ld8(taddr, r);
}
template <int N>
__device__ __forceinline__ void tmem_stn(uint32_t taddr, const uint32_t (&r)[N]) {
  if constexpr (N == 16) tmem_st16(taddr, r);
  else tmem_st8(taddr, r);
}

// PERSISTENT: CTA c runs items cta_items[cta_off[c] .. cta_off[c+1]) back to back (host LPT plan);
// the X~ ring, the S / P double buffers and their barriers run across items, U (by TMA) and O^T are
// double-buffered per item, so the next item's first tiles load and multiply while this item's
// sums are reduced and its outputs written.
template <bool STD, int NQ>
__global__ void __launch_bounds__(NCfg<NQ>::THREADS, 1)
    k_tc_attention_narrow(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapU,
                          const AttnItem *__restrict__ items, const int32_t *__restrict__ cta_off,
                          const int32_t *__restrict__ cta_items, bf16 *__restrict__ Y, float *__restrict__ part,
                          int yh) {
  // yh = 1: the reordered form -- an item's U rows and keys are whole rows of U [N_t h x d] and X~.
  // yh = h: the STANDARD form (Eq.(12), stca_set_attention_form): U [N_t x h d] holds per head r the query
  // q W_Q^r (zero-padded to d columns) and the keys are K/V rows [T' x h d] holding [K^r | V^r | 0] per
  // head; item.pad = r selects the 128-column block of both, and the output row of query t is t h + r.
  using C = NCfg<NQ>;
  constexpr int CW = C::CW;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *sX = smem;
  uint8_t *sP = sX + C::STAGES * C::X_BYTES;
  uint8_t *sU = sP + 2 * C::P_BYTES;                                   // 2 buffers
  float *sRed = reinterpret_cast<float *>(sU + 2 * C::U_BYTES);        // [4][4][16]
  float *sDefL = sRed + 4 * 4 * CW;                                    // [4][4][CW] deferred item's partial sums
  float *sDefM = sDefL + 4 * 4 * CW;                                   // [4][CW] deferred item's maxima
  // (both only with C::DEFER: DEF_BYTES is 0 otherwise)
  uint32_t *sFlag = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(sRed) + C::RED_BYTES + C::DEF_BYTES);
  uint64_t *bar = reinterpret_cast<uint64_t *>(sFlag + 16);
  uint64_t *u_full = bar;                      // 2 (TMA)
  uint64_t *u_free = u_full + 2;               // 2 (S issuer commit after an item's last S)
  uint64_t *x_full = u_free + 2;               // STAGES
  uint64_t *x_empty = x_full + C::STAGES;      // STAGES (PV commit)
  uint64_t *s_full = x_empty + C::STAGES;      // 2
  uint64_t *s_free = s_full + 2;               // 2 (NSW warps)
  uint64_t *p_full = s_free + 2;               // 2 (NSW warps)
  uint64_t *pv_done = p_full + 2;              // 2
  uint64_t *o_free = pv_done + 2;              // 2 (NSW warps: O^T buffer read out)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(o_free + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int i0 = cta_off[blockIdx.x], i1 = cta_off[blockIdx.x + 1];
  if (C::RESERVE == 0 && (smem_u32(smem_raw) & 1023) != 0) __trap();  // no room to align (see NCfg)

  if (warp == C::NSW && lane == 0) {
    tma_prefetch(&mapX);
    tma_prefetch(&mapU);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&u_full[b], 1);
      mbar_init(&u_free[b], 1);
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], C::NSW);
      mbar_init(&p_full[b], C::NSW);
      mbar_init(&pv_done[b], 1);
      mbar_init(&o_free[b], C::NSW);
    }
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&x_full[s], 1);
      mbar_init(&x_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == C::NSW + 1) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();  // U comes from the preceding GEMM (programmatic dependent launch)
  pdl_trigger();

  if (warp == C::NSW) {
    if (lane == 0) {  // ---------------- TMA producer: per item U, then its key tiles ----------------
      int s = 0, ph = 0;
      // L2 prefetch cursor, STCA_NARROW_PF key tiles ahead of the loads, across item boundaries
      int pf_n = i0, pf_j = 0, pf_nt = 0, pf_col = 0;
      int64_t pf_key0 = 0;
      if (i0 < i1) {
        const AttnItem f = items[cta_items[i0]];
        pf_nt = (f.klen + C::BK - 1) / C::BK;
        pf_key0 = f.key0;
        pf_col = STD ? C::D * f.pad : 0;
      }
      auto pf_step = [&]() {  // prefetch the tile under the cursor, then advance it
        if (pf_n >= i1) return;
        const int32_t row = (int32_t)(pf_key0 + (int64_t)pf_j * C::BK);
        tma_prefetch_l2(&mapX, pf_col, row);
        tma_prefetch_l2(&mapX, pf_col + 64, row);
        if (++pf_j >= pf_nt) {
          pf_j = 0;
          if (++pf_n < i1) {
            const AttnItem f = items[cta_items[pf_n]];
            pf_nt = (f.klen + C::BK - 1) / C::BK;
            pf_key0 = f.key0;
            pf_col = STD ? C::D * f.pad : 0;
          }
        }
      };
      for (int k = 0; k < STCA_NARROW_PF; ++k) pf_step();
      for (int n = i0; n < i1; ++n) {
        const AttnItem it = items[cta_items[n]];
        STCA_DCHECK(it.klen >= 1 && it.nq >= 1 && it.nq <= C::NQ && it.key0 >= 0 && it.qrow0 >= 0);
        const int ni = n - i0, ub = ni & 1, nt = (it.klen + C::BK - 1) / C::BK;
        if (ni >= 2) mbar_wait(&u_free[ub], ((ni - 2) >> 1) & 1);
        mbar_expect_tx(&u_full[ub], C::U_BYTES);
        uint8_t *ud = sU + ub * C::U_BYTES;
        const int32_t col0 = STD ? C::D * it.pad : 0;  // head block (standard form)
        tma_load_2d(ud, &mapU, &u_full[ub], col0, (int32_t)it.qrow0);  // rows past nq: finite, unused columns
        tma_load_2d(ud + C::U_BYTES / 2, &mapU, &u_full[ub], col0 + 64, (int32_t)it.qrow0);
        for (int j = 0; j < nt; ++j) {
          if (STCA_NARROW_PF > 0) pf_step();
          mbar_wait(&x_empty[s], ph ^ 1);
          uint8_t *dst = sX + s * C::X_BYTES;
          const int32_t row = (int32_t)(it.key0 + (int64_t)j * C::BK);
          mbar_expect_tx(&x_full[s], C::X_BYTES);
          tma_load_2d(dst, &mapX, &x_full[s], col0, row);
          tma_load_2d(dst + C::X_BYTES / 2, &mapX, &x_full[s], col0 + 64, row);
          if (++s == C::STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == C::NSW + 1) {
    if (lane == 0) {  // ---------------- S issuer: S^T_j = X~_j U^T (SS, M = 128, N = 64) ----------------
      constexpr uint32_t idesc_s = idesc_bf16(128, C::NQ, 0);
      const uint32_t aX = smem_u32(sX);
      int s = 0, ph = 0, g = 0;
      for (int n = i0; n < i1; ++n) {
        const AttnItem it = items[cta_items[n]];
        const int ni = n - i0, ub = ni & 1, nt = (it.klen + C::BK - 1) / C::BK;
        const uint32_t aU = smem_u32(sU + ub * C::U_BYTES);
        mbar_wait(&u_full[ub], (ni >> 1) & 1);
        for (int j = 0; j < nt; ++j, ++g) {
          const int b = g & 1;
          mbar_wait(&x_full[s], ph);
          if (g >= 2) mbar_wait(&s_free[b], ((g - 2) >> 1) & 1);
          tc_fence_after();
          const uint32_t xs = aX + s * C::X_BYTES;
#pragma unroll
          for (int k = 0; k < C::D / 16; ++k)
            umma_f16_ss(tmem + C::TS + b * C::NQ, sdesc_sw128(xs + (k >> 2) * (C::X_BYTES / 2) + (k & 3) * 32, 16, 1024),
                        sdesc_sw128(aU + (k >> 2) * (C::U_BYTES / 2) + (k & 3) * 32, 16, 1024), idesc_s, k != 0);
          umma_commit(&s_full[b]);
          if (++s == C::STAGES) { s = 0; ph ^= 1; }
        }
        umma_commit(&u_free[ub]);  // this item's U buffer may be reloaded
      }
    }
  } else if (warp == C::NSW + 2) {
    if (lane == 0) {  // ---------------- PV issuer: O^T += X~_j^T P_j^T (SS, both MN-major) ----------------
      constexpr uint32_t idesc_o = idesc_bf16_mn(128, C::NQ);
      const uint32_t aX = smem_u32(sX), aP = smem_u32(sP);
      int s = 0, g = 0;
      for (int n = i0; n < i1; ++n) {
        const AttnItem it = items[cta_items[n]];
        const int ni = n - i0, ob = ni & 1, nt = (it.klen + C::BK - 1) / C::BK;
        if (ni >= 2) mbar_wait(&o_free[ob], ((ni - 2) >> 1) & 1);  // O^T buffer ob read out (item ni - 2)
        for (int j = 0; j < nt; ++j, ++g) {
          const int b = g & 1;
          mbar_wait(&p_full[b], (g >> 1) & 1);  // P^T_j written (and O^T rescaled, if it had to be)
          tc_fence_after();
          const uint32_t xs = aX + s * C::X_BYTES, ps = aP + b * C::P_BYTES;
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k) {  // 16 keys per MMA: 2 swizzle atoms of 8 key rows
            const uint64_t bd = NQ == 64 ? sdesc_sw128(ps + k * 2048, C::P_BYTES, 1024)  // P^T rows of 128 B
                                         : sdesc_sw64(ps + k * 1024, C::P_BYTES, 512);   // P^T rows of 64 B
            umma_f16_ss(tmem + C::TO + ob * C::NQ, sdesc_sw128(xs + k * 2048, C::X_BYTES / 2, 1024), bd, idesc_o,
                        (j | k) != 0);
          }
          umma_commit(&pv_done[b]);
          umma_commit(&x_empty[s]);
          if (++s == C::STAGES) s = 0;
        }
      }
    }
  } else {  // ---------------- softmax warps 0..NSW-1 ----------------
    const int q = warp & 3, cg = warp >> 2;  // lane quarter (keys / d rows), 16-column query group
    const int key = q * 32 + lane;           // S^T lane = key within the tile; O^T lane = d
    const uint32_t lanes = (uint32_t)(q * 32) << 16;
    int g = 0;
    // DEFERRED epilogue: an item's output is written during the NEXT item's first tile (after its P is
    // handed to the PV issuer), so the softmax warps neither wait for the item's last PV nor hold up the
    // next item's pipeline start; the item's partial sums / maxima wait in sDefL / sDefM
    bool dpend = false;
    int dob = 0, dg = 0;  // deferred item's O^T buffer and last global tile
    AttnItem dit{};
    auto deferred_epilogue = [&]() {
      mbar_wait(&pv_done[dg & 1], (dg >> 1) & 1);  // the deferred item's last PV
      tc_fence_after();
      uint32_t o[CW];
      tmem_ldn<CW>(tmem + lanes + C::TO + dob * C::NQ + CW * cg, o);  // thread = output column d, CW queries
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[dob]);  // the PV issuer may start item + 2 in this buffer
      const int d = key;
#pragma unroll
      for (int e = 0; e < CW; ++e) {
        const int qn = CW * cg + e;
        if (qn < dit.nq) {
          const float ln = sDefL[(cg * 4) * CW + e] + sDefL[(cg * 4 + 1) * CW + e] + sDefL[(cg * 4 + 2) * CW + e] +
                           sDefL[(cg * 4 + 3) * CW + e];
          const bf16 y = __float2bfloat16(__uint_as_float(o[e]) / ln);
          if (dit.part_row < 0) {
            if constexpr (STD) Y[((dit.qrow0 + qn) * yh + dit.pad) * C::D + d] = y;
            else Y[(dit.qrow0 + qn) * C::D + d] = y;
          } else {  // partials hold the chunk's normalised output O / l, then (m, l)
            uint8_t *pr = reinterpret_cast<uint8_t *>(part) + (dit.part_row + qn) * (int64_t)part_row_bytes(C::D, 2);
            reinterpret_cast<bf16 *>(pr)[d] = y;
            if (d == 0) *reinterpret_cast<float2 *>(pr + 2 * C::D) = make_float2(sDefM[cg * CW + e], ln);
          }
        }
      }
      dpend = false;
    };
    for (int n = i0; n < i1; ++n) {
      const AttnItem it = items[cta_items[n]];
      const int ni = n - i0, ob = ni & 1, nt = (it.klen + C::BK - 1) / C::BK;
      float mref[CW], l[CW];
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        mref[c] = -INFINITY;
        l[c] = 0.f;
      }
      for (int j = 0; j < nt; ++j, ++g) {
        const int b = g & 1;
        mbar_wait(&s_full[b], (g >> 1) & 1);
        tc_fence_after();
        uint32_t sr[CW];
        tmem_ldn<CW>(tmem + lanes + C::TS + b * C::NQ + CW * cg, sr);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[b]);
        const bool kv = key < it.klen - j * C::BK;
        float dm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < CW; ++c) dm[c & 3] = fmaxf(dm[c & 3], __uint_as_float(sr[c]) - mref[c]);
        const bool need = kv && fmaxf(fmaxf(dm[0], dm[1]), fmaxf(dm[2], dm[3])) > STCA_NARROW_LAZY;
        const uint32_t wneed = __any_sync(0xffffffffu, need);
        uint8_t *flags = reinterpret_cast<uint8_t *>(sFlag + 4 * b + cg);
        if (lane == 0) flags[q] = (uint8_t)wneed;
        named_bar_sync(1 + cg, 128);
        if (*reinterpret_cast<volatile uint32_t *>(flags) != 0) {  // column maxima of this key tile (rare)
          float v[CW];
#pragma unroll
          for (int c = 0; c < CW; ++c) v[c] = kv ? __uint_as_float(sr[c]) : -INFINITY;
          const float red = xreduce<true, CW>(v, lane);
          if (lane < CW) sRed[(cg * 4 + q) * CW + lane] = red;
          named_bar_sync(1 + cg, 128);
          float f[CW];
          bool any = false;
#pragma unroll
          for (int c = 0; c < CW; c += 4) {
            float4 t = *reinterpret_cast<const float4 *>(sRed + (cg * 4) * CW + c);
#pragma unroll
            for (int qq = 1; qq < 4; ++qq) {
              const float4 u = *reinterpret_cast<const float4 *>(sRed + (cg * 4 + qq) * CW + c);
              t = make_float4(fmaxf(t.x, u.x), fmaxf(t.y, u.y), fmaxf(t.z, u.z), fmaxf(t.w, u.w));
            }
            const float tm[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const bool up = tm[e] > mref[c + e] + STCA_NARROW_LAZY;
              f[c + e] = up ? ex2(mref[c + e] - tm[e]) : 1.f;  // 0 for the first maximum (-inf reference)
              any |= up && j > 0;
              if (up) mref[c + e] = tm[e];
            }
          }
#pragma unroll
          for (int c = 0; c < CW; ++c) l[c] *= f[c];
          if (__any_sync(0xffffffffu, any)) {  // rescale O^T columns once the PVs issued so far are done
            mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
            tc_fence_after();
            uint32_t o[CW];
            tmem_ldn<CW>(tmem + lanes + C::TO + ob * C::NQ + CW * cg, o);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < CW; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f[c]);
            tmem_stn<CW>(tmem + lanes + C::TO + ob * C::NQ + CW * cg, o);
            tmem_st_wait();
          }
        }
        // the exponentials on MUFU; an A/B build puts the first C::NFMA of the thread's CW on the FMA pipe
        // (packed cubic, ex2_fma2, relative error 1e-4)
        uint32_t w[CW / 2];
#pragma unroll
        for (int i = 0; i < CW / 2; ++i) {
          const float x0 = __uint_as_float(sr[2 * i]) - mref[2 * i], x1 = __uint_as_float(sr[2 * i + 1]) - mref[2 * i + 1];
          float p0, p1;
          if (2 * i < C::NFMA) {
            const uint64_t e2 = ex2_fma2(f2_pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f)));
            p0 = kv ? f2_lo(e2) : 0.f;
            p1 = kv ? f2_hi(e2) : 0.f;
          } else {
            p0 = kv ? ex2(x0) : 0.f;
            p1 = kv ? ex2(x1) : 0.f;
          }
          l[2 * i] += p0;
          l[2 * i + 1] += p1;
          w[i] = pack_bf16(p0, p1);
        }
        if (g >= 2) mbar_wait(&pv_done[b], ((g - 2) >> 1) & 1);  // PV of tile g-2 has read P^T buffer b
        uint8_t *prow = sP + b * C::P_BYTES;
#pragma unroll
        for (int k = 0; k < CW / 8; ++k)
          *reinterpret_cast<uint4 *>(prow + (NQ == 64 ? sw128_off(key, 2 * cg + k) : sw64_off(key, cg))) =
              make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
        fence_proxy_async();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
        if (C::DEFER && dpend) deferred_epilogue();  // the previous item's output (first tile of this item only)
      }
      if constexpr (C::DEFER) {
        // ---- sums over the keys: per warp by recursive halving; the 4 lane quarters are added by the
        // deferred epilogue (sDefL survives this item's successor's first tile, which reuses sRed) ----
        if (nt == 1) named_bar_sync(1 + cg, 128);  // the deferred epilogue in this (only) tile read sDefL
        {
          const float red = xreduce<false, CW>(l, lane);
          if (lane < CW) sDefL[(cg * 4 + q) * CW + lane] = red;
          if (q == 0 && lane < CW) {
            float mv = mref[0];
#pragma unroll
            for (int c = 1; c < CW; ++c) mv = lane == c ? mref[c] : mv;
            sDefM[cg * CW + lane] = mv;
          }
        }
        dpend = true;
        dob = ob;
        dg = g - 1;
        dit = it;
      } else {
        // ---- sums over the keys: per warp by recursive halving, then the 4 lane quarters through SMEM ----
        named_bar_sync(1 + cg, 128);  // the last tile's sRed reads are done
        {
          const float red = xreduce<false, CW>(l, lane);
          if (lane < CW) sRed[(cg * 4 + q) * CW + lane] = red;
        }
        if (nt >= 1) mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);  // the item's last PV
        tc_fence_before();
        named_bar_sync(1 + cg, 128);
        tc_fence_after();
        uint32_t o[CW];
        tmem_ldn<CW>(tmem + lanes + C::TO + ob * C::NQ + CW * cg, o);  // thread = output column d, CW queries
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_free[ob]);  // the PV issuer may start item ni + 2 in this buffer
        const int d = key;
#pragma unroll
        for (int e = 0; e < CW; ++e) {
          const int qn = CW * cg + e;
          if (qn < it.nq) {
            const float ln = sRed[(cg * 4) * CW + e] + sRed[(cg * 4 + 1) * CW + e] + sRed[(cg * 4 + 2) * CW + e] +
                             sRed[(cg * 4 + 3) * CW + e];
            const bf16 y = __float2bfloat16(__uint_as_float(o[e]) / ln);
            if (it.part_row < 0) {
              if constexpr (STD) Y[((it.qrow0 + qn) * yh + it.pad) * C::D + d] = y;
              else Y[(it.qrow0 + qn) * C::D + d] = y;
            } else {  // partials hold the chunk's normalised output O / l, then (m, l)
              uint8_t *pr = reinterpret_cast<uint8_t *>(part) + (it.part_row + qn) * (int64_t)part_row_bytes(C::D, 2);
              reinterpret_cast<bf16 *>(pr)[d] = y;
              if (d == 0) *reinterpret_cast<float2 *>(pr + 2 * C::D) = make_float2(mref[e], ln);
            }
          }
        }
      }
    }
    if (C::DEFER && dpend) {  // the CTA's last item
      named_bar_sync(1 + cg, 128);  // its sDefL / sDefM writes are visible to the column group
      deferred_epilogue();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == C::NSW + 1) tmem_dealloc(tmem, 256);
}

}  // namespace tc

bool tc_attention_narrow_supported(int d, int max_rows) { return d == 128 && max_rows <= 64; }

// ncols = 64 or 32: the query columns of the instantiation (a request with m_b h <= 32 takes the
// 32-column kernel: half the MMA N, the exponentials and the softmax registers of the 64-column one)
template <int NQ>
static cudaError_t narrow_launch(const void *U, int64_t NQrows, const void *Xt, int64_t T2, const AttnItem *items,
                                 const int32_t *cta_off, const int32_t *cta_items, int n_ctas, void *Y, float *part,
                                 cudaStream_t st, int yh) {
  using C = tc::NCfg<NQ>;
  CUtensorMap mx, mu;
  // standard form (yh = h): U is [N_t x h d], the keys [T' x h d]; an item reads one d-column block of each
  const int64_t cols = (int64_t)C::D * yh;
  if (!tc::make_map_bf16(&mx, Xt, T2, cols, cols, C::BK) || !tc::make_map_bf16(&mu, U, NQrows / yh, cols, cols, C::NQ))
    return cudaErrorInvalidValue;
  // separate instantiations: the standard form's per-item head offsets cost the reordered form registers
  // (spill loads 60 -> 316 bytes, +12-18 % at multi / train) when compiled into one kernel
  const void *kfn = yh > 1 ? (const void *)tc::k_tc_attention_narrow<true, NQ> : (const void *)tc::k_tc_attention_narrow<false, NQ>;
  cudaError_t e0 = smem_optin(kfn, C::SMEM);
  if (e0 != cudaSuccess) return e0;
  note_launch();
  if (yh > 1)
    return launch_pdl(tc::k_tc_attention_narrow<true, NQ>, dim3((unsigned)n_ctas), dim3(C::THREADS), (size_t)C::SMEM,
                      st, mx, mu, items, cta_off, cta_items, (bf16 *)Y, part, yh);
  return launch_pdl(tc::k_tc_attention_narrow<false, NQ>, dim3((unsigned)n_ctas), dim3(C::THREADS), (size_t)C::SMEM, st,
                    mx, mu, items, cta_off, cta_items, (bf16 *)Y, part, yh);
}

cudaError_t tc_attention_narrow(const void *U, int64_t NQ, const void *Xt, int64_t T2, const AttnItem *items,
                                const int32_t *cta_off, const int32_t *cta_items, int n_ctas, void *Y, float *part,
                                cudaStream_t st, int yh, int ncols) {
  if (n_ctas <= 0) return cudaSuccess;
  if (ncols == 32) return narrow_launch<32>(U, NQ, Xt, T2, items, cta_off, cta_items, n_ctas, Y, part, st, yh);
  if (ncols == 64) return narrow_launch<64>(U, NQ, Xt, T2, items, cta_off, cta_items, n_ctas, Y, part, st, yh);
  return cudaErrorInvalidValue;
}

}  // namespace stca
