// tc_attn.cu -- fused ragged single-query cross attention on tcgen05 (sm_100a).
//
// PAPER.md Eq.(13): per head r, u = (q W_Q^r) W_K^r^T, alpha = softmax(u X~^T /
// sqrt(d_h)), y = alpha X~.  Under RLB every target-head pair (t, r) of one
// request is one query row u_{t,r} (pre-scaled by log2(e)/sqrt(d_h)) against the SAME
// history rows X~_b, so a request's m_b*h query rows form the M side of two real MMAs:
//     S = U_b X~_b^T   (M = 128 query rows, N = 128 keys, K = d)
//     O += P X~_b      (M = 128, N = d, K = 128 keys)
// Ragged Target Attention: keys are the flattened [T' x d] cache; a work item
// covers one request's key chunk, keys past the chunk end are masked to -inf (P = 0).
//
// One SMEM copy of each X~ tile (TMA, SWIZZLE_128B, two 64-column boxes) is read by the
// first MMA as a K-major B operand and by the second as an MN-major B operand.  S is
// double-buffered in TMEM, O lives in TMEM; the softmax warps (one thread per query row)
// keep the running max / sum in fp32 registers, write P (bf16) into SMEM in the UMMA
// K-major SW128 layout, and rescale O only when the running max grows by more than
// 2^8 (exact: the final 1/l uses the same stale max).  Output: normalised Y (bf16) for
// single-chunk requests, or (max, sum, O) fp32 partials for the split-K merge.
//
// Warp roles (192 threads): 0..3 = softmax / correction / epilogue (TMEM lane quarter = warp),
// 4 = TMA producer, 5 = TMEM allocator + MMA issuer (highest ids: the warp arbiter prefers them).
#include <math.h>

#include "launch.h"
#include "tc.h"
#include "tc_ptx.cuh"

namespace stca {
namespace tc {

bool make_map_bf16(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

constexpr int AT_BM = 128;       // query rows per CTA
constexpr int AT_BN = 128;       // keys per tile
constexpr int AT_D = 128;        // head-input width d (= row width of X~)
constexpr int AT_STAGES = 3;     // X~ tile ring
constexpr int AT_U_BYTES = AT_BM * AT_D * 2;   // 32 KB
constexpr int AT_X_BYTES = AT_BN * AT_D * 2;   // 32 KB
constexpr int AT_P_BYTES = AT_BM * AT_BN * 2;  // 32 KB
constexpr int AT_SMEM = 1024 + AT_U_BYTES + AT_STAGES * AT_X_BYTES + 2 * AT_P_BYTES + 256;
constexpr float AT_RESCALE_THRESHOLD = 8.f;    // log2(256)

__global__ void __launch_bounds__(192, 1)
    k_tc_attention(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapX,
                   const AttnItem *__restrict__ items, bf16 *__restrict__ Y, float *__restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *sU = smem;
  uint8_t *sX = sU + AT_U_BYTES;
  uint8_t *sP = sX + AT_STAGES * AT_X_BYTES;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sP + 2 * AT_P_BYTES);
  uint64_t *u_full = bar;                  // 1
  uint64_t *x_full = bar + 1;              // AT_STAGES
  uint64_t *x_empty = x_full + AT_STAGES;  // AT_STAGES
  uint64_t *s_full = x_empty + AT_STAGES;  // 2
  uint64_t *p_full = s_full + 2;           // 2
  uint64_t *pv_done = p_full + 2;          // 2
  uint32_t *tslot = reinterpret_cast<uint32_t *>(pv_done + 2);

  const AttnItem it = items[blockIdx.x];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nt = (it.klen + AT_BN - 1) / AT_BN;

  if (warp == 4 && lane == 0) {
    tma_prefetch(&mapU);
    tma_prefetch(&mapX);
    mbar_init(u_full, 1);
    for (int s = 0; s < AT_STAGES; ++s) {
      mbar_init(&x_full[s], 1);
      mbar_init(&x_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 128);
      mbar_init(&pv_done[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tO = tmem + 256;  // S buffers at cols [0,128) and [128,256); O at [256,384)

  if (warp == 4) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      const uint64_t pol_x = policy_evict_first();
      mbar_expect_tx(u_full, AT_U_BYTES);
      tma_load_2d(sU, &mapU, u_full, 0, (int32_t)it.qrow0);
      tma_load_2d(sU + AT_U_BYTES / 2, &mapU, u_full, 64, (int32_t)it.qrow0);
      for (int j = 0; j < nt; ++j) {
        const int s = j % AT_STAGES;
        mbar_wait(&x_empty[s], ((j / AT_STAGES) & 1) ^ 1);
        uint8_t *dst = sX + s * AT_X_BYTES;
        const int32_t row = (int32_t)(it.key0 + (int64_t)j * AT_BN);
        mbar_expect_tx(&x_full[s], AT_X_BYTES);
        tma_load_2d_hint(dst, &mapX, &x_full[s], 0, row, pol_x);
        tma_load_2d_hint(dst + AT_X_BYTES / 2, &mapX, &x_full[s], 64, row, pol_x);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc_s = idesc_bf16(AT_BM, AT_BN, 0);  // S = U X~^T : B K-major
      constexpr uint32_t idesc_o = idesc_bf16(AT_BM, AT_D, 1);   // O += P X~  : B MN-major
      const uint32_t aU = smem_u32(sU), aX = smem_u32(sX), aP = smem_u32(sP);
      mbar_wait(u_full, 0);
      auto pv = [&](int j) {  // O += P_j X~_j
        const int s = j % AT_STAGES, b = j & 1;
        mbar_wait(&p_full[b], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t xs = aX + s * AT_X_BYTES, ps = aP + b * AT_P_BYTES;
#pragma unroll
        for (int k = 0; k < AT_BN / 16; ++k) {
          const uint64_t ad = sdesc_sw128(ps + (k >> 2) * (AT_P_BYTES / 2) + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(xs + k * 2048, AT_X_BYTES / 2, 1024);  // MN-major: LBO = 64-col box
          umma_f16_ss(tO, ad, bd, idesc_o, (j | k) != 0);
        }
        umma_commit(&pv_done[b]);
        umma_commit(&x_empty[s]);
      };
      for (int j = 0; j < nt; ++j) {
        const int s = j % AT_STAGES, b = j & 1;
        mbar_wait(&x_full[s], (j / AT_STAGES) & 1);
        if (j >= 2) mbar_wait(&p_full[b], ((j - 2) >> 1) & 1);  // S buffer b consumed by softmax
        tc_fence_after();
        const uint32_t xs = aX + s * AT_X_BYTES;
#pragma unroll
        for (int k = 0; k < AT_D / 16; ++k) {
          const uint64_t ad = sdesc_sw128(aU + (k >> 2) * (AT_U_BYTES / 2) + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(xs + (k >> 2) * (AT_X_BYTES / 2) + (k & 3) * 32, 16, 1024);
          umma_f16_ss(tS + b * AT_BN, ad, bd, idesc_s, k != 0);
        }
        umma_commit(&s_full[b]);
        if (j >= 1) pv(j - 1);
      }
      if (nt >= 1) pv(nt - 1);
    }
  } else {  // ---------------- softmax / correction / epilogue ----------------
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nt; ++j) {
      const int b = j & 1;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
      const int kvalid = it.klen - j * AT_BN;  // keys of this tile that belong to the chunk
      uint32_t sr[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t (&r)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]);
        tmem_ld32(tS + lane_off + b * AT_BN + 32 * c, r);
      }
      tmem_ld_wait();
      float mt = -INFINITY;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        float v = c < kvalid ? __uint_as_float(sr[c]) : -INFINITY;
        sr[c] = __float_as_uint(v);
        mt = fmaxf(mt, v);
      }
      const bool need = mt > m + AT_RESCALE_THRESHOLD;
      if (j == 0) {
        m = mt;
      } else if (__any_sync(0xffffffffu, need)) {
        // warp-uniform (tcgen05.ld/st are .sync.aligned): O = O * 2^(m - m_new) per row once
        // every PV issued so far has landed; rows that do not need it use scale 1
        mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
        const float mnew = need ? mt : m;
        const float sc = exp2f(m - mnew);
        l *= sc;
#pragma unroll 1
        for (int c = 0; c < AT_D; c += 16) {
          uint32_t o[16];
          tmem_ld16(tO + lane_off + c, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * sc);
          tmem_st16(tO + lane_off + c, o);
        }
        tmem_st_wait();
        m = mnew;
      }
      // P = 2^(S - m) (bf16), row sum of the rounded values
      if (j >= 2) mbar_wait(&pv_done[b], ((j - 2) >> 1) & 1);  // MMA of tile j-2 done reading P buffer b
      uint8_t *pb = sP + b * AT_P_BYTES;
      float ls = 0.f;
#pragma unroll
      for (int c8 = 0; c8 < 16; ++c8) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float p0 = ex2(__uint_as_float(sr[8 * c8 + 2 * i]) - m);
          const float p1 = ex2(__uint_as_float(sr[8 * c8 + 2 * i + 1]) - m);
          w[i] = pack_bf16(p0, p1);
          __nv_bfloat162 h2 = *reinterpret_cast<__nv_bfloat162 *>(&w[i]);
          ls += __low2float(h2) + __high2float(h2);
        }
        const uint32_t off = (c8 >> 3) * (AT_P_BYTES / 2) + sw128_off(row, c8 & 7);
        *reinterpret_cast<uint4 *>(pb + off) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      l += ls;
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&p_full[b]);
    }
    // epilogue: wait for the last PV, then write Y = O / l or the (m, l, O) partial
    if (nt >= 1) mbar_wait(&pv_done[(nt - 1) & 1], ((nt - 1) >> 1) & 1);
    tc_fence_after();
    const bool ok = row < it.nq;
    if (it.part_row < 0) {
      const float inv = 1.f / l;
      bf16 *yr = Y + (it.qrow0 + row) * AT_D;
#pragma unroll 1
      for (int c = 0; c < AT_D; c += 32) {
        uint32_t o[32];
        tmem_ld32(tO + lane_off + c, o);
        tmem_ld_wait();
        if (ok) {
          uint4 *dst = reinterpret_cast<uint4 *>(yr + c);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16(__uint_as_float(o[8 * i]) * inv, __uint_as_float(o[8 * i + 1]) * inv),
                                pack_bf16(__uint_as_float(o[8 * i + 2]) * inv, __uint_as_float(o[8 * i + 3]) * inv),
                                pack_bf16(__uint_as_float(o[8 * i + 4]) * inv, __uint_as_float(o[8 * i + 5]) * inv),
                                pack_bf16(__uint_as_float(o[8 * i + 6]) * inv, __uint_as_float(o[8 * i + 7]) * inv));
        }
      }
    } else {
      float *pr = part + (it.part_row + row) * (int64_t)(AT_D + 2);
      if (ok) {
        pr[0] = m;
        pr[1] = l;
      }
#pragma unroll 1
      for (int c = 0; c < AT_D; c += 32) {
        uint32_t o[32];
        tmem_ld32(tO + lane_off + c, o);
        tmem_ld_wait();
        if (ok) {
#pragma unroll
          for (int i = 0; i < 32; i += 2)
            *reinterpret_cast<float2 *>(pr + 2 + c + i) = make_float2(__uint_as_float(o[i]), __uint_as_float(o[i + 1]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc(tmem, 512);
}

}  // namespace tc

bool tc_attention_supported(int d) { return d == tc::AT_D; }

cudaError_t tc_attention(const void *U, int64_t NQ, const void *Xt, int64_t T2, const AttnItem *items,
                         int64_t n_items, int d, void *Y, float *part, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  if (d != tc::AT_D) return cudaErrorInvalidValue;
  // U is [NQ x d]: query-tile rows past NQ are zero-filled by TMA (and never written back)
  CUtensorMap mu, mx;
  if (!tc::make_map_bf16(&mu, U, NQ, d, d, 128) || !tc::make_map_bf16(&mx, Xt, T2, d, d, 128))
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc::k_tc_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::AT_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  note_launch();
  tc::k_tc_attention<<<(unsigned)n_items, 192, tc::AT_SMEM, st>>>(mu, mx, items, (bf16 *)Y, part);
  return cudaGetLastError();
}

}  // namespace stca
