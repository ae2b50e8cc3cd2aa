// tc_attn_pair.cu -- ragged single-query attention for wide histories (d = 256, 512) on CTA PAIRS
// (tcgen05 cta_group::2), SURVEY §2.2 K-C at the capacity shape.
//
// Same computation as tc_attn.cu (Eq.(13); Ragged Target Attention):
// per request, S = U_b X~_b^T, P = 2^(S - m), Y = P X~_b / sum, U pre-scaled by log2(e)/sqrt(d_h).
//
// Why pairs.  At d = 512 a 128-row fp32 output tile alone fills all 512 TMEM columns, so one CTA
// can only run M = 64 MMAs -- which cost an M = 128 MMA's cycles (half rate).  A cta_group::2 MMA of
// M = 128 gives each CTA of a cluster pair 64 query rows at FULL rate, and its accumulator takes only
// N/2 TMEM columns per CTA: rows 0-63 in lanes 0-63 with the first N/2 columns, the same rows in
// lanes 64-127 with the last N/2 columns (measured: tools/pair_m128_layout.cu).  Per CTA:
//   TMEM  O [64 rows x d] = d/2 columns (two N = 256 MMAs at d = 512) | S [64 x 64 keys] x 2 buffers
//   SMEM  U [64 rows x d] (the SS A operand of S; a TMEM A operand would have to be replicated in
//         both lane halves, measured, leaving no room for S) | X~ ring | P [64 x 64] x 2 buffers
// The leader CTA (rank 0) issues every MMA for the pair; B operands are split between the CTAs:
//   S  = U X~_j^T:  N = 64 keys, CTA r holds keys [32 r, 32 r + 32) of the tile x all d (K-major)
//   PV: O += P X~_j: per d half h, N = 256, CTA r holds d columns [256 h + 128 r, + 128) x all 64
//       keys (MN-major)
// so each CTA loads 64 KB per 64-key tile at d = 512 (the two parts overlap by 16 KB: the shared
// descriptor needs the same SMEM offsets in both CTAs).  Key tiles are also prefetched into L2 ahead
// of the ring.  Softmax: TMEM lane L holds row L % 64 and keys [32 (L / 64), + 32); the two halves
// of a row exchange their maxima through SMEM (one 64-thread named barrier per tile) and keep a
// LAZY reference maximum (rescale O only when a tile's maximum exceeds it by > 2^8, as in
// tc_attn_wide.cu).  One pair per work item (request, 128 query rows, key chunk).
#include <math.h>

#include "launch.h"
#include "tc.h"
#include "tc_ptx.cuh"

#ifndef STCA_PAIR_LAZY
#define STCA_PAIR_LAZY 8.f  // rescale threshold in log2 units (a test build sets 0)
#endif
#ifndef STCA_PAIR_PF
#define STCA_PAIR_PF 3  // key tiles prefetched into L2 ahead of the loads
#endif

namespace stca {
namespace tc {

bool make_map_bf16(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

template <int D>
struct PCfg {
  static constexpr int BN = 64;                       // keys per tile
  static constexpr int NB = D / 64;                   // 64-column d blocks
  static constexpr int NPV = D / 256;                 // PV MMAs of N = 256
  static constexpr int BOX = 32 * 128;                // [32 keys x 64 d] SW128 box, 4 KB
  static constexpr int S_BYTES = NB * BOX;            // this CTA's 32 keys x all d
  static constexpr int PV_BYTES = NPV * 2 * 2 * BOX;  // all 64 keys x this CTA's 2 NPV d blocks
  // two rings with different lifetimes: an S part is free once S(j) is done (early), a PV part once
  // PV(j) is done; so the S-part loads of tile j + SS start long before the PV parts are needed
  static constexpr int SS = D == 512 ? 2 : 4, PS = D == 512 ? 2 : 4;
  static constexpr int U_BYTES = NB * 8192;           // 64 rows x d: NB boxes of [64 x 64]
  static constexpr int P_BYTES = 64 * 64 * 2;         // [64 rows x 64 keys] bf16, SW128 K-major
  // S and P buffers: 3 each, so the leader issues S two tiles ahead of PV (S(j), then PV(j - 2)) and the
  // softmax of a tile has two tiles of tensor work to hide behind
  static constexpr int NSB = 3, LA = NSB - 1;
  static constexpr int SMEM = 1024 + SS * S_BYTES + PS * PV_BYTES + U_BYTES + NSB * P_BYTES + 6 * 128 * 4 + 2 * 64 * 4 + 256;
  static constexpr uint32_t TO = 0, TS = 256;         // TMEM columns: O (NPV x 128) | S0 | S1 (32 each)
  static constexpr int THREADS = 352;  // warps 0-7 softmax (0-3) / output, 8 TMA (S parts), 9 MMA, 10 TMA (PV parts)
};

template <int D>
__global__ void __launch_bounds__(352, 1)
    k_tc_attention_pair(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapU,
                        const AttnItem *__restrict__ items, bf16 *__restrict__ Y, float *__restrict__ part) {
  using C = PCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *sXs = smem;                           // S-part ring
  uint8_t *sXp = sXs + C::SS * C::S_BYTES;       // PV-part ring
  uint8_t *sU = sXp + C::PS * C::PV_BYTES;
  uint8_t *sP = sU + C::U_BYTES;
  float *sXm = reinterpret_cast<float *>(sP + C::NSB * C::P_BYTES);  // [2 buf][2 col half][128 lane] tile maxima | [2][128] sums
  float *sMl = sXm + 6 * 128;                                    // [2][64]: reference maximum, total sum per row
  uint64_t *bar = reinterpret_cast<uint64_t *>(sMl + 2 * 64);
  uint64_t *sfull = bar;                    // SS (leader: S-part TMA bytes of both CTAs)
  uint64_t *sempty = sfull + C::SS;         // SS (commit multicast: S of the slot's tile done)
  uint64_t *pfull2 = sempty + C::SS;        // PS (leader: PV-part TMA bytes of both CTAs)
  uint64_t *pempty = pfull2 + C::PS;        // PS (commit multicast: PV of the slot's tile done)
  uint64_t *u_full = pempty + C::PS;        // 1 (leader: U bytes of both CTAs)
  uint64_t *s_full = u_full + 1;            // NSB (commit multicast)
  // (no "S buffer free" barrier: S(j + NSB) is issued after PV(j + 1 - ...) -- after PV(j), which waited
  // for P(j), so the softmax has long read S(j))
  uint64_t *p_full = s_full + C::NSB;       // NSB (leader: one arrive per CTA once its P half is written)
  uint64_t *pv_done = p_full + C::NSB;      // NSB (commit multicast)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(pv_done + C::NSB);

  const AttnItem it = items[blockIdx.x >> 1];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int nt = (it.klen + C::BN - 1) / C::BN;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&mapX);
    tma_prefetch(&mapU);
    for (int s = 0; s < C::SS; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 1);
    }
    for (int s = 0; s < C::PS; ++s) {
      mbar_init(&pfull2[s], 1);
      mbar_init(&pempty[s], 1);
    }
    mbar_init(u_full, 1);
    for (int b = 0; b < C::NSB; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 2);
      mbar_init(&pv_done[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc_pair(tslot, 512);
  tc_fence_before();
  cluster_sync_all();  // barrier inits visible pair-wide before any remote arrive / TMA completion
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();  // U comes from the preceding GEMM
  pdl_trigger();

  if (warp == 8) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs): U, then the key tiles ----------------
      const uint64_t pol = policy_evict_first();
      const uint32_t fb_u = mapa_shared(u_full, 0);
      if (rank == 0) mbar_expect_tx(u_full, 2 * C::U_BYTES);
#pragma unroll
      for (int b = 0; b < C::NB; ++b)
        tma_load_2d_pair(sU + b * 8192, &mapU, fb_u, 64 * b, (int32_t)(it.qrow0 + 64 * rank), policy_evict_normal());
      int pf = 0;
      auto prefetch = [&](int j) {  // both key halves, all d blocks of tile j (each CTA: its S half)
        if (j >= nt) return;
        const int32_t row = (int32_t)(it.key0 + (int64_t)j * C::BN + 32 * rank);
#pragma unroll
        for (int b = 0; b < C::NB; ++b) tma_prefetch_l2(&mapX, 64 * b, row);
      };
      for (; pf < STCA_PAIR_PF; ++pf) prefetch(pf);
      int s = 0, ph = 0;
      for (int j = 0; j < nt; ++j) {  // S parts: this CTA's 32 keys x all d
        prefetch(pf++);
        mbar_wait(&sempty[s], ph ^ 1);
        const uint32_t fb = mapa_shared(&sfull[s], 0);
        if (rank == 0) mbar_expect_tx(&sfull[s], 2 * C::S_BYTES);
        const int32_t k0 = (int32_t)(it.key0 + (int64_t)j * C::BN);
#pragma unroll
        for (int b = 0; b < C::NB; ++b)
          tma_load_2d_pair(sXs + s * C::S_BYTES + b * C::BOX, &mapX, fb, 64 * b, k0 + 32 * (int32_t)rank, pol);
        if (++s == C::SS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 10) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs): the PV parts ----------------
      const uint64_t pol = policy_evict_first();
      int s = 0, ph = 0;
      for (int j = 0; j < nt; ++j) {  // all 64 keys x d blocks 4h + 2 rank + jj
        mbar_wait(&pempty[s], ph ^ 1);
        const uint32_t fb = mapa_shared(&pfull2[s], 0);
        if (rank == 0) mbar_expect_tx(&pfull2[s], 2 * C::PV_BYTES);
        const int32_t k0 = (int32_t)(it.key0 + (int64_t)j * C::BN);
#pragma unroll
        for (int h = 0; h < C::NPV; ++h)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            uint8_t *pv = sXp + s * C::PV_BYTES + (2 * h + jj) * 2 * C::BOX;
            const int32_t c0 = 64 * (4 * h + 2 * (int32_t)rank + jj);
            tma_load_2d_pair(pv, &mapX, fb, c0, k0, pol);
            tma_load_2d_pair(pv + C::BOX, &mapX, fb, c0, k0 + 32, pol);
          }
        if (++s == C::PS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 9) {
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer of the pair (leader) ----------------
      constexpr uint32_t idesc_s = idesc_bf16(128, C::BN, 0);   // B K-major
      constexpr uint32_t idesc_o = idesc_bf16(128, 256, 1);     // B MN-major
      const uint32_t aXs = smem_u32(sXs), aXp = smem_u32(sXp), aU = smem_u32(sU), aP = smem_u32(sP);
      mbar_wait(u_full, 0);
      int s = 0, ph = 0, sp = 0, pph = 0;  // ring slots of S(j) and of PV(j - 1)
      auto issue_pv = [&](int j) {
        const int b = j % C::NSB;
        mbar_wait(&p_full[b], (j / C::NSB) & 1);
        mbar_wait(&pfull2[sp], pph);
        tc_fence_after();
        const uint32_t xs = aXp + sp * C::PV_BYTES, ps = aP + b * C::P_BYTES;
#pragma unroll
        for (int k = 0; k < C::BN / 16; ++k) {
          const uint64_t ad = sdesc_sw128(ps + k * 32, 16, 1024);
#pragma unroll
          for (int h = 0; h < C::NPV; ++h)
            umma_f16_ss_pair(tmem + C::TO + h * 128, ad, sdesc_sw128(xs + h * 4 * C::BOX + k * 2048, 2 * C::BOX, 1024),
                             idesc_o, (j | k) != 0);
        }
        umma_commit_pair_mc(&pv_done[b], 0x3);
        umma_commit_pair_mc(&pempty[sp], 0x3);
        if (++sp == C::PS) { sp = 0; pph ^= 1; }
      };
      for (int j = 0; j < nt; ++j) {
        const int b = j % C::NSB;
        mbar_wait(&sfull[s], ph);
        tc_fence_after();
        const uint32_t xs = aXs + s * C::S_BYTES;
#pragma unroll 8
        for (int k = 0; k < D / 16; ++k)
          umma_f16_ss_pair(tmem + C::TS + b * 32, sdesc_sw128(aU + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024),
                           sdesc_sw128(xs + (k >> 2) * C::BOX + (k & 3) * 32, 16, 1024), idesc_s, k != 0);
        umma_commit_pair_mc(&s_full[b], 0x3);
        umma_commit_pair_mc(&sempty[s], 0x3);
        if (++s == C::SS) { s = 0; ph ^= 1; }
        if (j >= C::LA) issue_pv(j - C::LA);  // S(j) and S(j - 1) run while the softmax of tile j - LA finishes
      }
      for (int j = nt > C::LA ? nt - C::LA : 0; j < nt; ++j) issue_pv(j);
    }
  } else {  // ---------------- warps 0-7: softmax and output ----------------
    // warp w: TMEM lane quarter q = w % 4, S column half ch = w / 4.  Thread: lane L = 32 q + lane holds
    // row r = L % 64, keys [32 hf + 16 ch, + 16) of the tile (hf = L / 64); a row's four partial maxima
    // (hf, ch) meet in shared memory at one 256-thread barrier per tile
    const int q = warp & 3, ch = warp >> 2;
    const int L = q * 32 + lane, r = L & 63, hf = L >> 6;
    const uint32_t lanes = (uint32_t)(q * 32) << 16;
    uint32_t pfull_b[C::NSB];
#pragma unroll
    for (int i = 0; i < C::NSB; ++i) pfull_b[i] = mapa_shared(&p_full[i], 0);
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < nt; ++j) {
      const int b = j % C::NSB;
      mbar_wait(&s_full[b], (j / C::NSB) & 1);
      tc_fence_after();
      uint32_t sr[16];
      tmem_ld16(tmem + lanes + C::TS + b * 32 + 16 * ch, sr);
      tmem_ld_wait();
      const int kvalid = it.klen - j * C::BN - 32 * hf - 16 * ch;
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < kvalid) mx[c & 3] = fmaxf(mx[c & 3], __uint_as_float(sr[c]));
      float tm = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      float *xm = sXm + (j & 1) * 256;  // two buffers suffice: every thread passes two barriers between uses
      xm[ch * 128 + L] = tm;
      named_bar_sync(1, 256);
      tm = fmaxf(fmaxf(tm, xm[(ch ^ 1) * 128 + L]), fmaxf(xm[ch * 128 + (L ^ 64)], xm[(ch ^ 1) * 128 + (L ^ 64)]));
      if (j == 0) {
        m_ref = tm;  // tile 0 always holds a valid key of the item
      } else {
        const bool need = tm > m_ref + STCA_PAIR_LAZY;  // identical for the row's four threads
        if (__any_sync(0xffffffffu, need)) {  // rescale this lane's half of the O columns once the PVs so far are done
          mbar_wait(&pv_done[(j - 1) % C::NSB], ((j - 1) / C::NSB) & 1);
          tc_fence_after();
          const float f = need ? ex2(m_ref - tm) : 1.f;
          if (need) {
            l *= f;
            m_ref = tm;
          }
#pragma unroll 1
          for (int h = 0; h < C::NPV; ++h)
#pragma unroll 1
            for (int c = 0; c < 64; c += 32) {
              uint32_t o[32];
              tmem_ld32(tmem + lanes + C::TO + h * 128 + 64 * ch + c, o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
              tmem_st32(tmem + lanes + C::TO + h * 128 + 64 * ch + c, o);
            }
          tmem_st_wait();
        }
      }
      if (j >= C::NSB) mbar_wait(&pv_done[b], ((j - C::NSB) / C::NSB) & 1);  // PV of tile j - NSB has read P buffer b
      uint32_t w[8];
      float lsum = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float p0 = 2 * i < kvalid ? ex2(__uint_as_float(sr[2 * i]) - m_ref) : 0.f;
        const float p1 = 2 * i + 1 < kvalid ? ex2(__uint_as_float(sr[2 * i + 1]) - m_ref) : 0.f;
        w[i] = pack_bf16(p0, p1);
        lsum += p0 + p1;
      }
      l += lsum;
      uint8_t *prow = sP + b * C::P_BYTES;
      *reinterpret_cast<uint4 *>(prow + sw128_off(r, 4 * hf + 2 * ch)) = make_uint4(w[0], w[1], w[2], w[3]);
      *reinterpret_cast<uint4 *>(prow + sw128_off(r, 4 * hf + 2 * ch + 1)) = make_uint4(w[4], w[5], w[6], w[7]);
      fence_proxy_async();
      tc_fence_before();
      named_bar_sync(2, 256);  // this CTA's P half is written: one cluster-scope arrive for all of it
      if (warp == 0 && lane == 0) mbar_arrive_cluster(pfull_b[b]);
    }
    // the row's total sum: its four partial sums
    float *sl = sXm + 4 * 128;
    sl[ch * 128 + L] = l;
    if (nt >= 1) mbar_wait(&pv_done[(nt - 1) % C::NSB], ((nt - 1) / C::NSB) & 1);  // the last PV
    tc_fence_before();
    named_bar_sync(1, 256);
    tc_fence_after();
    if (hf == 0 && ch == 0) {
      sMl[r] = m_ref;
      sMl[64 + r] = (sl[L] + sl[128 + L]) + (sl[L ^ 64] + sl[128 + (L ^ 64)]);
    }
    named_bar_sync(1, 256);
    // ---- output: warp (q, cg = warp / 4): lane L's O columns [128 h + 64 cg, + 64) = d 256 h + 128 hf + 64 cg + ..
    const int cg = warp >> 2;
    const int qrow = 64 * (int)rank + r;
    const bool ok = qrow < it.nq;  // per lane: tcgen05.ld below stays warp-uniform, only the stores are predicated
    const float inv = 1.f / sMl[64 + r];
    const bool partial = it.part_row >= 0;
    uint8_t *prow = partial ? reinterpret_cast<uint8_t *>(part) + (it.part_row + qrow) * (int64_t)part_row_bytes(D, 2)
                            : reinterpret_cast<uint8_t *>(Y + (it.qrow0 + qrow) * D);
    if (ok && partial && hf == 0 && cg == 0) *reinterpret_cast<float2 *>(prow + 2 * D) = make_float2(sMl[r], sMl[64 + r]);
#pragma unroll 1
    for (int h = 0; h < C::NPV; ++h)
#pragma unroll 1
      for (int c = 0; c < 64; c += 32) {
        uint32_t o[32];
        tmem_ld32(tmem + lanes + C::TO + h * 128 + 64 * cg + c, o);
        tmem_ld_wait();
        if (ok) {
          uint4 *dst = reinterpret_cast<uint4 *>(prow + 2 * (256 * h + 128 * hf + 64 * cg + c));
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16(__uint_as_float(o[8 * i]) * inv, __uint_as_float(o[8 * i + 1]) * inv),
                                pack_bf16(__uint_as_float(o[8 * i + 2]) * inv, __uint_as_float(o[8 * i + 3]) * inv),
                                pack_bf16(__uint_as_float(o[8 * i + 4]) * inv, __uint_as_float(o[8 * i + 5]) * inv),
                                pack_bf16(__uint_as_float(o[8 * i + 6]) * inv, __uint_as_float(o[8 * i + 7]) * inv));
        }
      }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer no longer arrives on / multicasts into this CTA
  if (warp == 9) tmem_dealloc_pair(tmem, 512);
}

}  // namespace tc

bool tc_attention_pair_supported(int d) { return d == 256 || d == 512; }

cudaError_t tc_attention_pair(const void *U, int64_t NQ, const void *Xt, int64_t T2, const AttnItem *items,
                              int64_t n_items, int d, void *Y, float *part, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  CUtensorMap mx, mu;
  if (!tc::make_map_bf16(&mx, Xt, T2, d, d, 32) || !tc::make_map_bf16(&mu, U, NQ, d, d, 64)) return cudaErrorInvalidValue;
#define PLAUNCH(DD)                                                                                            \
  {                                                                                                            \
    using C = tc::PCfg<DD>;                                                                                    \
    cudaError_t e0 = smem_optin((const void *)tc::k_tc_attention_pair<DD>, C::SMEM);                           \
    if (e0 != cudaSuccess) return e0;                                                                          \
    note_launch();                                                                                             \
    cudaLaunchConfig_t cfg = {};                                                                               \
    cfg.gridDim = dim3((unsigned)(2 * n_items));                                                               \
    cfg.blockDim = dim3(C::THREADS);                                                                           \
    cfg.dynamicSmemBytes = C::SMEM;                                                                            \
    cfg.stream = st;                                                                                           \
    cudaLaunchAttribute attr[2];                                                                               \
    attr[0].id = cudaLaunchAttributeClusterDimension;                                                          \
    attr[0].val.clusterDim.x = 2;                                                                              \
    attr[0].val.clusterDim.y = 1;                                                                              \
    attr[0].val.clusterDim.z = 1;                                                                              \
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                           \
    attr[1].val.programmaticStreamSerializationAllowed = 1;                                                    \
    cfg.attrs = attr;                                                                                          \
    cfg.numAttrs = 2;                                                                                          \
    cudaError_t e = cudaLaunchKernelEx(&cfg, tc::k_tc_attention_pair<DD>, mx, mu, items, (bf16 *)Y, part);     \
    return e != cudaSuccess ? e : cudaGetLastError();                                                          \
  }
  if (d == 512) PLAUNCH(512)
  if (d == 256) PLAUNCH(256)
#undef PLAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace stca
