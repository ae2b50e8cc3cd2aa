// tc_attn.cu -- fused ragged single-query cross attention on tcgen05 (sm_100a), SURVEY §2.2 K-C.
//
// PAPER.md Eq.(13): per head r, u = (q W_Q^r) W_K^r^T, alpha = softmax(u X~^T /
// sqrt(d_h)), y = alpha X~.  Under RLB every target-head pair (t, r) of one request
// is one query row u_{t,r} (pre-scaled by log2(e)/sqrt(d_h)) against the SAME history rows X~_b,
// so a request's m_b*h query rows form the M side of two real MMAs:
//     S = U_b X~_b^T   (M = 128 query rows, N = 128 keys, K = d)
//     O += P X~_b      (M = 128, N = d, K = 128 keys)
// Ragged Target Attention: keys are the flattened [T' x d] cache; a work item covers
// one request's key chunk, keys past the chunk end are masked to -inf (P = 0).
//
// PERSISTENT: one CTA per SM walks a host-planned list of work items (LPT bins, stca_plan_persistent),
// so the next item's U tile and first X~ tiles are fetched while the current item still runs, and
// an item's epilogue overlaps the next item's first S MMAs.  TMEM: S 2 x 128 | O 128 | U 2 x 64.
// U arrives by TMA (SW128, into the SMEM area that the epilogue later stages its output in) and the
// softmax warps move it into TMEM U[k & 1] before the previous item's epilogue.  U and P live in
// TENSOR MEMORY and are the A operands of both MMAs (TS form); P is written by the softmax warps as
// packed bf16 over the first half of the very S columns it was computed from.  X~ tiles arrive by
// TMA (two 64-column SW128 boxes, 4-stage ring) and ONE shared-memory copy is read as the K-major B
// of S and as the MN-major B of PV.  The softmax keeps max / sum in fp32 registers and rescales O
// only when a row max grows by more than 2^8 (exact: the final 1/l uses the same stale max),
// warp-uniformly (tcgen05.ld/st are .sync.aligned).  Output: normalised Y (bf16) for single-chunk
// requests, else fp32 partials [O(d) | m | l | pad 2] for the split-K merge, both staged in SMEM
// and written with fully coalesced 16-byte stores (a row per thread straight to global touched 32
// sectors per store instruction).
//
// Warp roles (32 (4 NP + 3) threads, NP = 2): 0..4NP-1 softmax / correction / epilogue (TMEM lane
// quarter = warp % 4, key-column part = warp / 4: NP threads per query row exchange their maxima
// through shared memory), then the TMA producer, the TMEM allocator + S issuer and the PV issuer.
// Issuers get the highest warp ids (the SM's arbiter prefers them) and S / PV are issued from
// different warps so that one warp's mbarrier waits are covered by the other's queued MMAs.  Two
// tcgen05.commits per key tile (S done, PV done): the S issuer, which waits for PV anyway before
// reusing an S buffer, frees the X~ ring slot with a plain arrive (each commit costs the tensor
// pipe ~45 cycles, tools/mma_bench).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "launch.h"
#include "tc.h"
#include "tc_ptx.cuh"

namespace stca {
namespace tc {

bool make_map_bf16(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

constexpr int AT_BM = 128;                     // query rows per item
constexpr int AT_BN = 128;                     // keys per tile
constexpr int AT_D = 128;                      // head-input width d (= row width of X~)
constexpr int AT_STAGES = 4;                   // X~ tile ring
constexpr int AT_X_BYTES = AT_BN * AT_D * 2;   // 32 KB
constexpr int AT_U_BYTES = AT_BM * AT_D * 2;   // 32 KB (two SW128 boxes)
constexpr int AT_NP = 2;                       // key-column parts per query row (threads per row)
constexpr int AT_CW = AT_BN / AT_NP;           // key columns (and O columns) per softmax thread
constexpr int AT_NSW = 4 * AT_NP;              // softmax warps
constexpr int AT_YSTRIDE = AT_D * 2 + 16;      // staged output row (bytes): Y, or a partial row O/l | m | l | pad
constexpr int AT_STAGE_BYTES = AT_BM * AT_YSTRIDE;  // 34 KB epilogue staging; the next U tile lands at its start
constexpr int AT_MAXI = 128;                  // work items of a CTA cached in shared memory
constexpr int AT_SMEM = 1024 + AT_STAGES * AT_X_BYTES + AT_STAGE_BYTES + AT_MAXI * (int)sizeof(AttnItem) + 256;
constexpr float AT_RESCALE_THRESHOLD = 8.f;    // log2(256)
#ifndef STCA_ATTN_PF
#define STCA_ATTN_PF 4  // key tiles prefetched into L2 ahead of the TMA loads (0: off)
#endif
constexpr int AT_WP = AT_NSW, AT_WS = AT_NSW + 1, AT_WO = AT_NSW + 2, AT_THREADS = 32 * (AT_NSW + 3);
constexpr uint32_t AT_TS = 0, AT_TO = 256, AT_TU = 384;  // TMEM columns: S0 | S1 | O | U0 | U1

__global__ void __launch_bounds__(AT_THREADS, 1)
    k_tc_attention(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapU,
                   const AttnItem *__restrict__ items, const int32_t *__restrict__ cta_off,
                   const int32_t *__restrict__ cta_items, bf16 *__restrict__ Y, float *__restrict__ part,
                   unsigned long long *trace) {
#define AT_TR(slot)                                                 \
  do {                                                              \
    if (trace && blockIdx.x == 0 && (slot) < 8192) trace[(slot)] = clock64(); \
  } while (0)
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *sX = smem;
  uint8_t *sStage = sX + AT_STAGES * AT_X_BYTES;  // epilogue staging; the next U tile lands at its start
  AttnItem *sItem = reinterpret_cast<AttnItem *>(sStage + AT_STAGE_BYTES);  // this CTA's first AT_MAXI items
  uint64_t *bar = reinterpret_cast<uint64_t *>(sItem + AT_MAXI);
  uint64_t *x_full = bar;                    // AT_STAGES (TMA tx)
  uint64_t *x_empty = x_full + AT_STAGES;    // AT_STAGES (S issuer: PV of the slot's tile done)
  uint64_t *s_full = x_empty + AT_STAGES;    // 2 (S MMA done)
  uint64_t *p_full = s_full + 2;             // 2 (softmax warps: P written into TMEM)
  uint64_t *pv_done = p_full + 2;            // 2 (PV MMA done: P / S buffer free, O stable)
  uint64_t *us_full = pv_done + 2;           // 1 (TMA tx: next U tile in SMEM)
  uint64_t *us_free = us_full + 1;           // 1 (softmax warps: U copied to TMEM; the staging area is free)
  uint64_t *u_full = us_free + 1;            // 2 (softmax warps: U[k & 1] in TMEM)
  uint64_t *o_free = u_full + 2;             // 1 (softmax warps: O read by the epilogue)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(o_free + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int i0 = cta_off[blockIdx.x], ni = cta_off[blockIdx.x + 1] - i0;  // this CTA's items

  if (warp == AT_WP && lane == 0) {
    tma_prefetch(&mapX);
    tma_prefetch(&mapU);
    for (int s = 0; s < AT_STAGES; ++s) {
      mbar_init(&x_full[s], 1);
      mbar_init(&x_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], AT_NSW);
      mbar_init(&pv_done[b], 1);
      mbar_init(&u_full[b], AT_NSW);
    }
    mbar_init(us_full, 1);
    mbar_init(us_free, AT_NSW);
    mbar_init(o_free, AT_NSW);
    fence_mbar_init();
  }
  if (warp == AT_WS) tmem_alloc(tslot, 512);
  pdl_wait();     // the predecessor's outputs (U) are complete and visible
  pdl_trigger();
  for (int k = threadIdx.x; k < ni && k < AT_MAXI; k += blockDim.x) sItem[k] = items[cta_items[i0 + k]];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // item k's descriptor: shared memory (the dependent global loads cost ~1500 cycles per item)
  auto item = [&](int k) -> AttnItem { return k < AT_MAXI ? sItem[k] : items[cta_items[i0 + k]]; };

  if (warp == AT_WP) {
    if (lane == 0) {  // ---------------- TMA producer: U tiles and the X~ ring ----------------
      const uint64_t pol_x = policy_evict_first();
      int s = 0, ph = 0;
      // L2 prefetch cursor, STCA_ATTN_PF key tiles ahead of the loads, across item boundaries
      int pf_k = 0, pf_j = 0, pf_nt = 0;
      int64_t pf_key0 = 0;
      if (ni > 0) {
        const AttnItem f = item(0);
        pf_nt = (f.klen + AT_BN - 1) / AT_BN;
        pf_key0 = f.key0;
      }
      auto pf_step = [&]() {
        if (pf_k >= ni) return;
        const int32_t row = (int32_t)(pf_key0 + (int64_t)pf_j * AT_BN);
        tma_prefetch_l2(&mapX, 0, row);
        tma_prefetch_l2(&mapX, 64, row);
        if (++pf_j >= pf_nt) {
          pf_j = 0;
          if (++pf_k < ni) {
            const AttnItem f = item(pf_k);
            pf_nt = (f.klen + AT_BN - 1) / AT_BN;
            pf_key0 = f.key0;
          }
        }
      };
      for (int k = 0; k < STCA_ATTN_PF; ++k) pf_step();
      for (int k = 0; k < ni; ++k) {
        const AttnItem it = item(k);
        STCA_DCHECK(it.klen >= 1 && it.nq >= 1 && it.nq <= AT_BM && it.key0 >= 0 && it.qrow0 >= 0);
        // U of item k into the staging area once the softmax warps moved U(k-1) into TMEM and the
        // epilogue of item k-2 (which staged its output there) is done; both are one us_free phase
        if (k >= 1) mbar_wait(us_free, (k - 1) & 1);
        mbar_expect_tx(us_full, AT_U_BYTES);
        tma_load_2d(sStage, &mapU, us_full, 0, (int32_t)it.qrow0);
        tma_load_2d(sStage + AT_U_BYTES / 2, &mapU, us_full, 64, (int32_t)it.qrow0);
        const int nt = (it.klen + AT_BN - 1) / AT_BN;
        for (int j = 0; j < nt; ++j) {
          if (STCA_ATTN_PF > 0) pf_step();
          mbar_wait(&x_empty[s], ph ^ 1);
          uint8_t *dst = sX + s * AT_X_BYTES;
          const int32_t row = (int32_t)(it.key0 + (int64_t)j * AT_BN);
          mbar_expect_tx(&x_full[s], AT_X_BYTES);
          tma_load_2d_hint(dst, &mapX, &x_full[s], 0, row, pol_x);
          tma_load_2d_hint(dst + AT_X_BYTES / 2, &mapX, &x_full[s], 64, row, pol_x);
          if (++s == AT_STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == AT_WS) {
    if (lane == 0) {  // ---------------- S issuer: S_j = U X~_j^T ----------------
      constexpr uint32_t idesc_s = idesc_bf16(AT_BM, AT_BN, 0);  // B K-major
      const uint32_t aX = smem_u32(sX);
      int s = 0, ph = 0, jj = 0, sp = 0;  // ring slot, global tile counter, slot of tile jj - 2
      for (int k = 0; k < ni; ++k) {
        const AttnItem it = item(k);
        const int nt = (it.klen + AT_BN - 1) / AT_BN;
        mbar_wait(&u_full[k & 1], (k >> 1) & 1);
        const uint32_t tu = tmem + AT_TU + (k & 1) * 64;
        for (int j = 0; j < nt; ++j, ++jj) {
          const int b = jj & 1;
          if (jj >= 2) {  // PV_{jj-2} has read P from S buffer b and its X~ slot: free the slot first
            mbar_wait(&pv_done[b], ((jj - 2) >> 1) & 1);
            mbar_arrive(&x_empty[sp]);
            if (++sp == AT_STAGES) sp = 0;
          }
          AT_TR(jj * 16 + 1);
          mbar_wait(&x_full[s], ph);
          AT_TR(jj * 16 + 2);
          tc_fence_after();
          const uint32_t xs = aX + s * AT_X_BYTES;
#pragma unroll
          for (int kk = 0; kk < AT_D / 16; ++kk)
            umma_f16_ts(tmem + AT_TS + b * AT_BN, tu + kk * 8,
                        sdesc_sw128(xs + (kk >> 2) * (AT_X_BYTES / 2) + (kk & 3) * 32, 16, 1024), idesc_s, kk != 0);
          umma_commit(&s_full[b]);
          AT_TR(jj * 16 + 3);
          if (++s == AT_STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == AT_WO) {
    if (lane == 0) {  // ---------------- PV issuer: O += P_j X~_j ----------------
      constexpr uint32_t idesc_o = idesc_bf16(AT_BM, AT_D, 1);  // B MN-major
      const uint32_t aX = smem_u32(sX);
      int s = 0, jj = 0;
      for (int k = 0; k < ni; ++k) {
        const AttnItem it = item(k);
        const int nt = (it.klen + AT_BN - 1) / AT_BN;
        for (int j = 0; j < nt; ++j, ++jj) {
          const int b = jj & 1;
          mbar_wait(&p_full[b], (jj >> 1) & 1);
          if (j == 0 && k >= 1) mbar_wait(o_free, (k - 1) & 1);  // the previous item's epilogue read O
          AT_TR(jj * 16 + 4);
          tc_fence_after();
          const uint32_t xs = aX + s * AT_X_BYTES;
#pragma unroll
          for (int kk = 0; kk < AT_BN / 16; ++kk)
            umma_f16_ts(tmem + AT_TO, tmem + AT_TS + b * AT_BN + kk * 8,
                        sdesc_sw128(xs + kk * 2048, AT_X_BYTES / 2, 1024), idesc_o, (j | kk) != 0);
          umma_commit(&pv_done[b]);
          AT_TR(jj * 16 + 5);
          if (++s == AT_STAGES) s = 0;
        }
      }
    }
  } else {  // -------- softmax / correction / epilogue: AT_NSW warps, one row x AT_CW key columns each --------
    // 16x32bx2 TMEM access (tools/tmem_layout): warp w owns the 16 rows 32 (w % 4) + 16 (w / 4) + t of
    // its lane quarter; lane t < 16 and lane t + 16 share row t, holding key / O / U columns
    // [0, 64) and [64, 128) of it (pp = lane / 16).  The row max of a tile is one shuffle: the warps
    // never wait for each other inside a tile (no shared-memory exchange, no named barrier).
    const int pp = lane >> 4;
    const int row = (warp & 3) * 32 + (warp >> 2) * 16 + (lane & 15);
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32 + (warp >> 2) * 16) << 16;
    // U(k) (staged by TMA, SW128) -> TMEM U[k & 1] as packed bf16 pairs: this thread's 64 of d columns
    auto load_u = [&](int k) {
      mbar_wait(us_full, k & 1);
      const uint8_t *box = sStage + pp * (AT_U_BYTES / 2);  // pp = 64-column half of d
#pragma unroll
      for (int h16 = 0; h16 < 2; ++h16) {  // 32 bf16 = 16 packed columns per store
        uint32_t w[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint4 v = *reinterpret_cast<const uint4 *>(box + sw128_off(row, 4 * h16 + c));
          w[4 * c] = v.x;
          w[4 * c + 1] = v.y;
          w[4 * c + 2] = v.z;
          w[4 * c + 3] = v.w;
        }
        tmem_st16x2_16<32>(tmem + lane_off + AT_TU + (k & 1) * 64 + 16 * h16, w);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&u_full[k & 1]);
        if (k == 0) mbar_arrive(us_free);  // us_free phase 0: U(0) consumed; phase k >= 1: epilogue k-1 done
      }
    };
    if (ni > 0) load_u(0);
    int jj = 0;                 // global tile counter
    bool bulk_pending = false;  // warp 0: an item's output copy may still be reading the staging
    for (int k = 0; k < ni; ++k) {
      const AttnItem it = item(k);
      const int nt = (it.klen + AT_BN - 1) / AT_BN;
      float m = -INFINITY, l = 0.f;  // l: this thread's half of the row sum
      for (int j = 0; j < nt; ++j, ++jj) {
        const int b = jj & 1;
        mbar_wait(&s_full[b], (jj >> 1) & 1);
        if (warp == 0 && lane == 0) AT_TR(jj * 16 + 6);
        tc_fence_after();
        const int kvalid = it.klen - j * AT_BN - AT_CW * pp;  // keys of this half inside the chunk
        uint32_t sr[AT_CW];
        tmem_ld16x2_32<64>(tmem + lane_off + AT_TS + b * AT_BN, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        tmem_ld16x2_32<64>(tmem + lane_off + AT_TS + b * AT_BN + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        tmem_ld_wait();
        const bool partial = it.klen - j * AT_BN < AT_BN;  // warp-uniform: only a chunk's last tile is masked
        if (partial) {
#pragma unroll
          for (int c = 0; c < AT_CW; ++c)
            if (c >= kvalid) sr[c] = __float_as_uint(-INFINITY);
        }
        float mx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = -INFINITY;
#pragma unroll
        for (int c = 0; c < AT_CW; c += 2)
          mx[(c >> 1) & 7] = fmax3(mx[(c >> 1) & 7], __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
        float mt = fmaxf(fmaxf(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5])), fmaxf(mx[6], mx[7]));
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 16));  // the row's other half
        if (warp == 0 && lane == 0) AT_TR(jj * 16 + 7);
        const bool need = mt > m + AT_RESCALE_THRESHOLD;
        if (j == 0) {
          m = mt;
        } else if (__any_sync(0xffffffffu, need)) {
          // warp-uniform: O *= 2^(m - m_new) per row once every PV issued so far has landed
          mbar_wait(&pv_done[(jj - 1) & 1], ((jj - 1) >> 1) & 1);
          tc_fence_after();
          const float mnew = need ? mt : m;
          const float sc = exp2f(m - mnew);
          l *= sc;
#pragma unroll 1
          for (int c = 0; c < AT_CW; c += 16) {
            uint32_t o[16];
            tmem_ld16x2_16<64>(tmem + lane_off + AT_TO + c, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * sc);
            tmem_st16x2_16<64>(tmem + lane_off + AT_TO + c, o);
          }
          tmem_st_wait();
          m = mnew;
        }
        // P = 2^(S - m) as bf16 pairs: this thread's 64 keys -> S buffer b packed columns [32 pp, 32 pp + 32).
        // Packed fp32x2 arithmetic; on full tiles 3 of every 8 pairs of exponentials run on the FMA
        // pipe (ex2_fma2): at d = 128 one exp per (row, key) balances MUFU and the tensor pipe exactly.
        // The row sum accumulates the fp32 values.
        const uint64_t nm2 = f2_pack(-m, -m);
        uint64_t ls2[2] = {0ull, 0ull};
        uint32_t w[AT_CW / 2];
        if (partial) {  // masked keys must give exactly 0: MUFU ex2(-inf) = 0
#pragma unroll
          for (int i = 0; i < AT_CW / 2; ++i) {
            const uint64_t x2 = f2_add((uint64_t)sr[2 * i] | ((uint64_t)sr[2 * i + 1] << 32), nm2);
            const uint64_t e2 = f2_pack(ex2(f2_lo(x2)), ex2(f2_hi(x2)));
            w[i] = pack_bf16(f2_lo(e2), f2_hi(e2));
            ls2[i & 1] = f2_add(ls2[i & 1], e2);
          }
        } else {
#pragma unroll
          for (int i = 0; i < AT_CW / 2; ++i) {
            const uint64_t x2 = f2_add((uint64_t)sr[2 * i] | ((uint64_t)sr[2 * i + 1] << 32), nm2);
            uint64_t e2;
            if ((i & 7) == 1 || (i & 7) == 4 || (i & 7) == 6)
              e2 = ex2_fma2(f2_pack(fmaxf(f2_lo(x2), -126.f), fmaxf(f2_hi(x2), -126.f)));
            else
              e2 = f2_pack(ex2(f2_lo(x2)), ex2(f2_hi(x2)));
            w[i] = pack_bf16(f2_lo(e2), f2_hi(e2));
            ls2[i & 1] = f2_add(ls2[i & 1], e2);
          }
        }
        const uint64_t lsum = f2_add(ls2[0], ls2[1]);
        if (warp == 0 && lane == 0) AT_TR(jj * 16 + 12);
        tmem_st16x2_16<32>(tmem + lane_off + AT_TS + b * AT_BN, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
        tmem_st16x2_16<32>(tmem + lane_off + AT_TS + b * AT_BN + 16, *reinterpret_cast<uint32_t(*)[16]>(&w[16]));
        l += f2_lo(lsum) + f2_hi(lsum);
        tmem_st_wait();
        if (warp == 0 && lane == 0) AT_TR(jj * 16 + 13);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
        if (bulk_pending) {  // warp 0, first tile after an epilogue: the staging may take U(k+1) now
          bulk_wait_read0();
          __syncwarp();
          if (lane == 0) mbar_arrive(us_free);
          bulk_pending = false;
        }
        if (lane == 0 && (warp == 0 || warp == 4 || warp == AT_NSW - 1))
          AT_TR(jj * 16 + 9 + (warp == 0 ? 0 : warp == 4 ? 1 : 2));
      }
      // the next item's U into TMEM before this epilogue: its first S MMAs overlap the epilogue
#define AT_TRE(e) \
  if (warp == 0 && lane == 0 && k < 64) AT_TR(7680 + k * 8 + (e))
      AT_TRE(5);
      if (k + 1 < ni) load_u(k + 1);
      AT_TRE(6);
      // ---- epilogue: wait for the last PV, combine the parts' sums, stage, coalesced store ----
      mbar_wait(&pv_done[(jj - 1) & 1], ((jj - 1) >> 1) & 1);
      AT_TRE(0);
      tc_fence_after();
      const float lrow = l + __shfl_xor_sync(0xffffffffu, l, 16);  // the row's two halves
      named_bar_sync(1, 32 * AT_NSW);  // every warp is past its U copy: the staging area is free
      AT_TRE(1);
      const bool single = it.part_row < 0;
      const float inv = 1.f / lrow;
#pragma unroll 1
      for (int cb = 0; cb < AT_CW; cb += 32) {  // Y row, or the partial's normalised O / l (same bf16 form)
        uint32_t o[32];
        tmem_ld16x2_32<64>(tmem + lane_off + AT_TO + cb, o);
        tmem_ld_wait();
        uint8_t *dst = sStage + row * AT_YSTRIDE + (AT_CW * pp + cb) * 2;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          *reinterpret_cast<uint4 *>(dst + 16 * i) =
              make_uint4(pack_bf16(__uint_as_float(o[8 * i]) * inv, __uint_as_float(o[8 * i + 1]) * inv),
                         pack_bf16(__uint_as_float(o[8 * i + 2]) * inv, __uint_as_float(o[8 * i + 3]) * inv),
                         pack_bf16(__uint_as_float(o[8 * i + 4]) * inv, __uint_as_float(o[8 * i + 5]) * inv),
                         pack_bf16(__uint_as_float(o[8 * i + 6]) * inv, __uint_as_float(o[8 * i + 7]) * inv));
      }
      if (!single && pp == 0)
        *reinterpret_cast<float4 *>(sStage + row * AT_YSTRIDE + AT_D * 2) = make_float4(m, lrow, 0.f, 0.f);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_free);  // PV of the next item may overwrite O
      fence_proxy_async();                  // staged rows visible to the bulk copies below
      AT_TRE(2);
      named_bar_sync(1, 32 * AT_NSW);      // the item's rows are staged
      AT_TRE(3);
      // copy-out by the TMA engine (bulk copies, no registers): the item's nq output rows are
      // contiguous in global memory.  Warp 0 issues them; it confirms the staging has been read
      // (us_free) only after the next item's first tile, so no warp waits for the copy here.
      if (warp == 0) {
        if (single) {  // one 256-byte row per copy (the staging rows are padded)
          for (int r = lane; r < it.nq; r += 32)
            bulk_store(Y + (it.qrow0 + r) * AT_D, sStage + r * AT_YSTRIDE, AT_D * 2);
        } else if (lane == 0) {  // partial rows are contiguous with the staging's row stride
          bulk_store(reinterpret_cast<uint8_t *>(part) + it.part_row * AT_YSTRIDE, sStage, (uint32_t)it.nq * AT_YSTRIDE);
        }
        bulk_commit();
        bulk_pending = true;
      } else if (lane == 0) {
        mbar_arrive(us_free);  // this warp does not read the staging any more
      }
      AT_TRE(4);
#undef AT_TRE
    }
    if (bulk_pending) bulk_wait0();  // the last item's output written before the CTA exits
  }
  tc_fence_before();
  __syncthreads();
  if (warp == AT_WS) tmem_dealloc(tmem, 512);
}

}  // namespace tc

bool tc_attention_supported(int d) { return d == tc::AT_D; }
int tc_attention_ctas() { return sm_count(); }

cudaError_t tc_attention(const void *U, int64_t NQ, const void *Xt, int64_t T2, const AttnItem *items,
                         const int32_t *cta_off, const int32_t *cta_items, int n_ctas, int d, void *Y, float *part,
                         cudaStream_t st) {
  if (n_ctas <= 0) return cudaSuccess;
  if (d != tc::AT_D) return cudaErrorInvalidValue;
  CUtensorMap mx, mu;
  if (!tc::make_map_bf16(&mx, Xt, T2, d, d, 128) || !tc::make_map_bf16(&mu, U, NQ, d, d, 128))
    return cudaErrorInvalidValue;
  cudaError_t e0 = smem_optin((const void *)tc::k_tc_attention, tc::AT_SMEM);
  if (e0 != cudaSuccess) return e0;
  unsigned long long *trace = nullptr;
  const char *trace_path = getenv("STCA_TRACE_ATTN");  // debug only: clock64 stamps of CTA 0
  if (trace_path && cudaMalloc(&trace, 8192 * 8) == cudaSuccess) cudaMemsetAsync(trace, 0, 8192 * 8, st);
  note_launch();
  cudaError_t e = launch_pdl(tc::k_tc_attention, dim3((unsigned)n_ctas), dim3(tc::AT_THREADS), tc::AT_SMEM, st, mx, mu,
                             items, cta_off, cta_items, (bf16 *)Y, part, trace);
  if (e != cudaSuccess) return e;
  if (trace) {
    static unsigned long long h[8192];
    cudaMemcpyAsync(h, trace, sizeof h, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(trace);
    if (FILE *f = fopen(trace_path, "wb")) {
      fwrite(h, sizeof h, 1, f);
      fclose(f);
    }
  }
  return cudaGetLastError();
}

}  // namespace stca
