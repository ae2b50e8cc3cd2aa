// tc_attn_wide.cu -- ragged single-query attention for wide histories (d = 256, 512) on tcgen05.
//
// Same computation as tc_attn.cu (Eq.(13); Ragged Target Attention):
// per request, S = U_b X~_b^T, P = 2^(S - max), Y = P X~_b / sum, with U pre-scaled by
// log2(e)/sqrt(d_h).  At d = 512 an M = 128 output tile alone would fill all 512 TMEM columns, so
// this kernel works on 64 query rows with M = 64 MMAs, whose accumulator rows occupy 16 of the 32
// TMEM lanes of each warp quarter (measured: tools/m64_layout.cu, tools/m64_ts_check.cu):
//   lower lane half (lane base 0):  S double buffer (2 x 64 key columns) and U (the TMEM A operand
//                                   of S = U X~^T, d/2 packed columns)
//   upper lane half (lane base 16): O (d columns)
// P goes through shared memory (SW128 K-major) as the A operand of O += P X~ (SS mode; a TS
// operand must share the accumulator's lane half).  The softmax is ONE pass with a lazy running
// maximum: a row keeps its reference maximum m until a key tile's maximum exceeds it by more than
// 2^8 (P <= 256 is still exact enough in bf16 and the fp32 sums), and only then rescales its O row
// and l in place after the PV MMAs issued so far have completed — rare after the first tile, so
// S = U X~^T is computed once per key tile (the earlier two-pass form recomputed it: 3 MMA
// passes for 2 useful ones).  X~ tiles of 64 keys (d/64 boxes of 64 columns, 3-4 stage TMA ring)
// serve as the K-major B of S and the MN-major B of PV.
//
// Warp roles (352 threads): 0..3 softmax on the 16x32bx2 TMEM shape (threads t and t+16 share S
// row t of the warp's lane quarter, 32 key columns each; the row max is one shuffle) and O
// rescale; 0..7 load U and write the output (two warps per lane quarter, a quarter of the O
// columns each); 8 TMA producer, 9 TMEM allocator + S issuer, 10 PV issuer.
#include <math.h>

#include "launch.h"
#include "tc.h"
#include "tc_ptx.cuh"

#ifndef STCA_WIDE_LAZY
#define STCA_WIDE_LAZY 8.f  // rescale threshold in log2 units (a test build sets 0: rescale on every increase)
#endif
#ifndef STCA_WIDE_PF
#define STCA_WIDE_PF 4  // key tiles prefetched into L2 ahead of the TMA loads (0: off)
#endif

namespace stca {
namespace tc {

bool make_map_bf16(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

template <int D>
struct WCfg {
  static constexpr int BM = 64, BN = 64;                 // query rows, keys per tile
  static constexpr int X_BYTES = BN * D * 2;             // d/64 boxes of 64 x 64 (8 KB)
  static constexpr int STAGES = D == 512 ? 3 : 4;
  static constexpr int P_BYTES = BM * BN * 2;            // 8 KB, SW128 K-major
  static constexpr int SMEM = 1024 + STAGES * X_BYTES + 2 * P_BYTES + 2 * 64 * 4 + 256;
  static constexpr uint32_t TS = 0, TU = 256;            // lower lane half: S0 | S1 ... U
  static constexpr uint32_t TO = 16u << 16;              // upper lane half: O
};

template <int D>
__global__ void __launch_bounds__(352, 1)
    k_tc_attention_wide(const __grid_constant__ CUtensorMap mapX, const bf16 *__restrict__ U, int64_t NQ,
                        const AttnItem *__restrict__ items, bf16 *__restrict__ Y, float *__restrict__ part) {
  using C = WCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *sX = smem;
  uint8_t *sP = sX + C::STAGES * C::X_BYTES;
  float *sM = reinterpret_cast<float *>(sP + 2 * C::P_BYTES);  // [64] reference maximum per row
  float *sL = sM + 64;                                         // [64] sum per row
  uint64_t *bar = reinterpret_cast<uint64_t *>(sL + 64);
  uint64_t *u_full = bar;                      // 8 warp arrivals
  uint64_t *x_full = bar + 1;                  // STAGES
  uint64_t *x_empty = x_full + C::STAGES;      // STAGES (PV commit)
  uint64_t *s_full = x_empty + C::STAGES;      // 2
  uint64_t *s_free = s_full + 2;               // 2 (4 softmax warps)
  uint64_t *p_full = s_free + 2;               // 2 (4 softmax warps)
  uint64_t *pv_done = p_full + 2;              // 2
  uint32_t *tslot = reinterpret_cast<uint32_t *>(pv_done + 2);

  const AttnItem it = items[blockIdx.x];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nt = (it.klen + C::BN - 1) / C::BN;
  STCA_DCHECK(it.klen >= 1 && it.nq >= 1 && it.nq <= C::BM && it.key0 >= 0 && it.qrow0 >= 0);

  if (warp == 8 && lane == 0) {
    tma_prefetch(&mapX);
    mbar_init(u_full, 8);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&x_full[s], 1);
      mbar_init(&x_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 4);
      mbar_init(&p_full[b], 4);
      mbar_init(&pv_done[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 8) {
    if (lane == 0) {  // ---------------- TMA producer: the key tiles, once ----------------
      int s = 0, ph = 0;
      auto prefetch = [&](int j) {
        if (j >= nt) return;
#pragma unroll
        for (int bx = 0; bx < D / 64; ++bx) tma_prefetch_l2(&mapX, 64 * bx, (int32_t)(it.key0 + (int64_t)j * C::BN));
      };
      for (int j = 0; j < STCA_WIDE_PF; ++j) prefetch(j);
      for (int j = 0; j < nt; ++j) {
        if (STCA_WIDE_PF > 0) prefetch(j + STCA_WIDE_PF);
        mbar_wait(&x_empty[s], ph ^ 1);
        uint8_t *dst = sX + s * C::X_BYTES;
        const int32_t row = (int32_t)(it.key0 + (int64_t)j * C::BN);
        mbar_expect_tx(&x_full[s], C::X_BYTES);
#pragma unroll
        for (int bx = 0; bx < D / 64; ++bx) tma_load_2d(dst + bx * 8192, &mapX, &x_full[s], 64 * bx, row);
        if (++s == C::STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {  // ---------------- S issuer: S_j = U X~_j^T (TS, M = 64, N = 64) ----------------
      constexpr uint32_t idesc_s = idesc_bf16(64, C::BN, 0);
      const uint32_t aX = smem_u32(sX);
      mbar_wait(u_full, 0);
      int s = 0, ph = 0;
      for (int j = 0; j < nt; ++j) {
        const int b = j & 1;
        mbar_wait(&x_full[s], ph);
        if (j >= 2) mbar_wait(&s_free[b], ((j - 2) >> 1) & 1);
        tc_fence_after();
        const uint32_t xs = aX + s * C::X_BYTES;
#pragma unroll 8
        for (int k = 0; k < D / 16; ++k)
          umma_f16_ts(tmem + C::TS + b * C::BN, tmem + C::TU + k * 8,
                      sdesc_sw128(xs + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024), idesc_s, k != 0);
        umma_commit(&s_full[b]);
        if (++s == C::STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 10) {
    if (lane == 0) {  // ---------------- PV issuer: O += P_j X~_j (SS, M = 64, N <= 256) ----------------
      constexpr int NS = D < 256 ? D : 256;
      constexpr uint32_t idesc_o = idesc_bf16(64, NS, 1);
      const uint32_t aX = smem_u32(sX), aP = smem_u32(sP);
      int s = 0;
      for (int j = 0; j < nt; ++j) {
        const int b = j & 1;
        mbar_wait(&p_full[b], (j >> 1) & 1);  // P_j written (and O rescaled, if it had to be)
        tc_fence_after();
        const uint32_t xs = aX + s * C::X_BYTES, ps = aP + b * C::P_BYTES;
#pragma unroll
        for (int k = 0; k < C::BN / 16; ++k) {
          const uint64_t ad = sdesc_sw128(ps + k * 32, 16, 1024);
#pragma unroll
          for (int n = 0; n < D / NS; ++n)
            umma_f16_ss(tmem + C::TO + n * NS, ad, sdesc_sw128(xs + n * (NS / 64) * 8192 + k * 2048, 8192, 1024),
                        idesc_o, (j | k) != 0);
        }
        umma_commit(&pv_done[b]);
        umma_commit(&x_empty[s]);
        if (++s == C::STAGES) s = 0;
      }
    }
  } else {  // ---------------- warps 0..7: U load; 0..3 softmax; 0..7 output ----------------
    const int q = warp & 3, hh = warp >> 2;
    {  // U row -> TMEM lower half (the A operand of S); lanes 16-31 write zeros into the upper half
      const int r = q * 16 + (lane & 15);
      const int64_t grow = it.qrow0 + r;
      const bool ld = lane < 16 && grow < NQ;
      const uint4 *src = reinterpret_cast<const uint4 *>(U + grow * D + (D / 2) * hh);
      const uint32_t qoff = (uint32_t)(q * 32) << 16;
#pragma unroll
      for (int c = 0; c < D / 4; c += 16) {  // this half's D/2 bf16 = D/4 packed columns
        uint32_t w[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint4 v = ld ? src[(c / 16) * 4 + k] : make_uint4(0, 0, 0, 0);
          w[4 * k] = v.x;
          w[4 * k + 1] = v.y;
          w[4 * k + 2] = v.z;
          w[4 * k + 3] = v.w;
        }
        tmem_st16(tmem + qoff + C::TU + (D / 4) * hh + c, w);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(u_full);
    }
    // 16x32bx2 view of lane quarter q: thread t and t+16 <-> query row q*16 + (t & 15)
    const int pp = lane >> 4, r = q * 16 + (lane & 15);
    const uint32_t s_lanes = (uint32_t)(q * 32) << 16, o_lanes = (uint32_t)(q * 32 + 16) << 16;
    if (warp < 4) {
      float m_ref = -INFINITY, l = 0.f;  // identical in both threads of the row
      for (int j = 0; j < nt; ++j) {
        const int b = j & 1;
        mbar_wait(&s_full[b], (j >> 1) & 1);
        tc_fence_after();
        uint32_t sr[32];
        tmem_ld16x2_32<32>(tmem + s_lanes + C::TS + b * C::BN, sr);  // t: keys 0-31, t+16: keys 32-63
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[b]);
        const int kvalid = it.klen - j * C::BN - 32 * pp;
        float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c < kvalid) mx[c & 3] = fmaxf(mx[c & 3], __uint_as_float(sr[c]));
        float tm = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
        tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 16));
        if (j == 0) {
          m_ref = tm;  // tile 0 always holds a valid key of the item
        } else {
          const bool need = tm > m_ref + STCA_WIDE_LAZY;
          if (__any_sync(0xffffffffu, need)) {  // rescale this warp's O rows once the PVs so far are done
            mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
            tc_fence_after();
            const float f = need ? ex2(m_ref - tm) : 1.f;
            if (need) {
              l *= f;
              m_ref = tm;
            }
#pragma unroll 1
            for (int c = 0; c < D / 2; c += 32) {  // t: columns [c, c+32), t+16: [D/2 + c, D/2 + c + 32)
              uint32_t o[32];
              tmem_ld16x2_32<D / 2>(tmem + o_lanes + c, o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
              tmem_st16x2_32<D / 2>(tmem + o_lanes + c, o);
            }
            tmem_st_wait();
          }
        }
        const int pb = j & 1;
        if (j >= 2) mbar_wait(&pv_done[pb], ((j - 2) >> 1) & 1);  // PV of tile j-2 has read P buffer pb
        uint32_t w[16];
        float lsum = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p0 = 2 * i < kvalid ? ex2(__uint_as_float(sr[2 * i]) - m_ref) : 0.f;
          const float p1 = 2 * i + 1 < kvalid ? ex2(__uint_as_float(sr[2 * i + 1]) - m_ref) : 0.f;
          w[i] = pack_bf16(p0, p1);
          lsum += p0 + p1;
        }
        l += lsum;
        uint8_t *prow = sP + pb * C::P_BYTES;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          *reinterpret_cast<uint4 *>(prow + sw128_off(r, 4 * pp + k)) = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
        fence_proxy_async();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[pb]);
      }
      l += __shfl_xor_sync(0xffffffffu, l, 16);
      if (pp == 0) {
        sM[r] = m_ref;
        sL[r] = l;
      }
    }
    // the softmax warps (in step with pv_done) wait for the last PV; warps 4-7 would be phases ahead
    if (warp < 4 && nt >= 1) mbar_wait(&pv_done[(nt - 1) & 1], ((nt - 1) >> 1) & 1);
    tc_fence_before();
    named_bar_sync(1, 256);
    tc_fence_after();
    // ---- output: warp (q, hh) writes columns [hh D/4, (hh+1) D/4) (t) and D/2 + that (t+16) of its rows ----
    const float l = sL[r], inv = 1.f / l;
    const bool ok = r < it.nq;
#pragma unroll 1
    for (int c = hh * (D / 4); c < (hh + 1) * (D / 4); c += 32) {
      uint32_t o[32];
      tmem_ld16x2_32<D / 2>(tmem + o_lanes + c, o);
      tmem_ld_wait();
      if (ok) {
        const int col = c + pp * (D / 2);
        uint4 *dst;
        if (it.part_row < 0) {
          dst = reinterpret_cast<uint4 *>(Y + (it.qrow0 + r) * D + col);
        } else {  // partials hold the chunk's normalised output O / l, then (m, l)
          uint8_t *pr = reinterpret_cast<uint8_t *>(part) + (it.part_row + r) * (int64_t)part_row_bytes(D, 2);
          if (col == 0) *reinterpret_cast<float2 *>(pr + 2 * D) = make_float2(sM[r], l);
          dst = reinterpret_cast<uint4 *>(pr + 2 * col);
        }
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
  if (warp == 9) tmem_dealloc(tmem, 512);
}

}  // namespace tc

bool tc_attention_wide_supported(int d) { return d == 256 || d == 512; }

cudaError_t tc_attention_wide(const void *U, int64_t NQ, const void *Xt, int64_t T2, const AttnItem *items,
                              int64_t n_items, int d, void *Y, float *part, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  CUtensorMap mx;
  if (!tc::make_map_bf16(&mx, Xt, T2, d, d, 64)) return cudaErrorInvalidValue;
#define WLAUNCH(DD)                                                                                              \
  {                                                                                                              \
    cudaError_t e0 = smem_optin((const void *)tc::k_tc_attention_wide<DD>, tc::WCfg<DD>::SMEM);                 \
    if (e0 != cudaSuccess) return e0;                                                                            \
    note_launch();                                                                                               \
    tc::k_tc_attention_wide<DD><<<(unsigned)n_items, 352, tc::WCfg<DD>::SMEM, st>>>(mx, (const bf16 *)U, NQ, items, \
                                                                                     (bf16 *)Y, part);           \
    return cudaGetLastError();                                                                                   \
  }
  if (d == 512) WLAUNCH(512)
  if (d == 256) WLAUNCH(256)
#undef WLAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace stca
