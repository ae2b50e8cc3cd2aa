// tc_chain.cu -- the target-side update of one layer boundary as ONE tcgen05 kernel (d = 128),
// SURVEY §8(a) rows a5 -> a6 -> a3 (and a2 / a7):
//
//   o(i)   = [Y_r]_r W_VO(i)                                  Eq.(6) with Eq.(13)
//            -> Z[:, i] (fp32) and block i of the concatenation [x_t | o(1) | ... | o(M)] (bf16)
//   q(i+1) = SwiGLUFFN(i+1)([o(1) .. o(i) | x_t] W_C(i+1))     Eq.(7)
//   U(i+1) = q(i+1) W_QK(i+1)  (log2(e)/sqrt(d_h) folded in)   the reordered query
// or, at the stack's ends, q(1) = LN(SwiGLUFFN(1)(x_t)) -> U(1) (Eq.(3)) and o(M) -> z =
// SwiGLUFFN_Z([o(1..M) | x_t] W_Z) (Eq.(9)).  The unfused path ran each of these as its own GEMM
// launch (4-6 per layer, each latency-bound at N_t = 16384 rows: 11-17 us); here one CTA per 128
// target rows runs the whole chain with every intermediate (o, c, the SwiGLU hidden H, q) kept in
// TMEM / shared memory, and only the weights stream in (TMA ring, L2-resident).
//
//   stage o   A = Y rows (TMA)            B = W_VO^T (K = h d)      -> TMEM acc0 -> Z, ocat, SMEM T0
//   stage c   A = ocat blocks (TMA) + T0  B = W_C^T  (K = (i+1) d)  -> TMEM acc1 -> SMEM Tc
//   FFN1(k)   A = Tc                      B = W1 rows [128k, +128)  -> TMEM G[k&1] -> SwiGLU -> SMEM H[k&1]
//   FFN2(k)   A = H[k&1]                  B = Wo^T K-block k        -> TMEM acc0 (+=)  (one chunk behind FFN1)
//   q         acc0 (-> LayerNorm for q(1)) -> SMEM T0 (or z, fp32, at the last layer)
//   stage U   A = T0                      B = W_QK^T rows [128 j, +128) -> TMEM G[j&1] -> U (bf16)
//
// Warps: 0-7 epilogue (TMEM lane quarter = warp % 4, column half = warp / 4), 8 TMA producer,
// 9 TMEM allocator + MMA issuer.  Every box is [128 rows x 64 bf16] SW128 (16 KB); the ring of
// 16 KB slots carries A and B boxes in the exact order the issuer consumes them.
#include <math.h>

#include "launch.h"
#include "tc.h"
#include "tc_ptx.cuh"

namespace stca {
namespace tc {

bool make_map_bf16(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

enum { CH_FIRST = 0, CH_MID = 1, CH_LAST = 2 };

constexpr int CH_D = 128;
constexpr int CH_BOX = 128 * 64 * 2;  // 16 KB
constexpr int CH_SLOTS = 6;
constexpr int CH_THREADS = 320;
// SMEM: ring | T0 (o, later q) | Tc | H[2] | LN partials | barriers
constexpr int CH_SMEM = 1024 + CH_SLOTS * CH_BOX + 2 * CH_BOX + 2 * CH_BOX + 2 * CH_BOX + 2 * 128 * 8 + 512;
// TMEM columns
constexpr uint32_t CH_ACC0 = 0, CH_ACC1 = 128, CH_G0 = 256;  // G[b] at 256 + 128 b

struct ChainArgs {
  int mode, M, nkc, n_u, rd_chunks;  // nkc: K blocks of stage c; n_u: N blocks of U (h d / 128)
  int n_o_kb;                         // K blocks of stage o (h d / 64)
  int n_ocat_kb;                      // K blocks of stage c loaded from ocat (the rest is T0)
  int Nt;
  float *Z;                           // Z + (i - 1) d, row stride ldz
  int64_t ldz;
  bf16 *ocat;                         // + i d (the block o(i) goes to), row stride ldo
  int64_t ldo;
  bf16 *U;                            // [Nt x h d]
  int64_t ldu;
  float *zout;                        // [Nt x d] (CH_LAST with z)
  const float *g, *b;                 // LayerNorm of q(1)
  float eps;
  int do_o, do_c, do_u, do_z;
};

__device__ __forceinline__ float chain_swiglu(float u, float v) {  // u * silu(v) = a + a tanh(v / 2), a = u v / 2
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * v));
  const float a = 0.5f * u * v;
  return fmaf(a, t, a);
}

__global__ void __launch_bounds__(CH_THREADS, 1)
    k_tc_chain(const __grid_constant__ CUtensorMap mY, const __grid_constant__ CUtensorMap mOc,
               const __grid_constant__ CUtensorMap mWVO, const __grid_constant__ CUtensorMap mWC,
               const __grid_constant__ CUtensorMap mW1, const __grid_constant__ CUtensorMap mWo,
               const __grid_constant__ CUtensorMap mWQK, ChainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *ring = smem;
  uint8_t *T0 = ring + CH_SLOTS * CH_BOX;  // 2 boxes: o(i), later q
  uint8_t *Tc = T0 + 2 * CH_BOX;           // 2 boxes: c (or x_t)
  uint8_t *Hb = Tc + 2 * CH_BOX;           // H[2], one box each
  float2 *lnx = reinterpret_cast<float2 *>(Hb + 2 * CH_BOX);  // [2][128] (mean, M2) of each half row
  uint64_t *bar = reinterpret_cast<uint64_t *>(lnx + 2 * 128);
  uint64_t *full = bar, *empty = full + CH_SLOTS;
  uint64_t *acc_done = empty + CH_SLOTS;  // 1: o / c / q accumulators (in order; each commit one phase)
  uint64_t *g_done = acc_done + 1;        // 2: FFN1 chunk / U block in G[b]
  uint64_t *g_free = g_done + 2;          // 2: epilogue read G[b] (8 warps)
  uint64_t *h_ready = g_free + 2;         // 2: H[b] written (8 warps)
  uint64_t *h_free = h_ready + 2;         // 2: FFN2 read H[b] (commit)
  uint64_t *t_ready = h_free + 2;         // 1: T0 / Tc written (8 warps; in order: o, c, q)
  uint64_t *tc_tma = t_ready + 1;         // 1: x_t in Tc by TMA (CH_FIRST)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tc_tma + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int row0 = blockIdx.x * 128;

  if (warp == 8 && lane == 0) {
    for (const CUtensorMap *m : {&mY, &mOc, &mWVO, &mWC, &mW1, &mWo, &mWQK}) tma_prefetch(m);
    for (int s = 0; s < CH_SLOTS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_done, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&g_done[b], 1);
      mbar_init(&g_free[b], 8);
      mbar_init(&h_ready[b], 8);
      mbar_init(&h_free[b], 1);
    }
    mbar_init(t_ready, 8);
    mbar_init(tc_tma, 1);
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();  // Y / ocat / x_t come from the preceding kernels
  pdl_trigger();

  if (warp == 8) {
    if (lane == 0) {  // ---------------- TMA producer: boxes in the issuer's order ----------------
      int s = 0, ph = 0;
      auto load = [&](const CUtensorMap *m, int c0, int r0) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], CH_BOX);
        tma_load_2d(ring + s * CH_BOX, m, &full[s], c0, r0);
        if (++s == CH_SLOTS) { s = 0; ph ^= 1; }
      };
      if (a.mode == CH_FIRST) {  // x_t straight into Tc
        mbar_expect_tx(tc_tma, 2 * CH_BOX);
        tma_load_2d(Tc, &mOc, tc_tma, 0, row0);
        tma_load_2d(Tc + CH_BOX, &mOc, tc_tma, 64, row0);
      }
      if (a.do_o)
        for (int kb = 0; kb < a.n_o_kb; ++kb) {
          load(&mY, 64 * kb, row0);
          load(&mWVO, 64 * kb, 0);
        }
      if (a.do_c)
        for (int kb = 0; kb < a.nkc; ++kb) {
          if (kb < a.n_ocat_kb) load(&mOc, 64 * kb, row0);  // the rest of A is T0 (o(i), this kernel's)
          load(&mWC, 64 * kb, 0);
        }
      if (a.do_c || a.mode == CH_FIRST) {
        for (int k = 0; k <= a.rd_chunks; ++k) {
          if (k < a.rd_chunks) {  // FFN1(k): W1 rows [128 k, +128), K = d in two boxes
            load(&mW1, 0, 128 * k);
            load(&mW1, 64, 128 * k);
          }
          if (k >= 1) load(&mWo, 64 * (k - 1), 0);  // FFN2(k - 1)
        }
      }
      if (a.do_u)
        for (int j = 0; j < a.n_u; ++j) {
          load(&mWQK, 0, 128 * j);
          load(&mWQK, 64, 128 * j);
        }
    }
  } else if (warp == 9) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = idesc_bf16(128, 128, 0);
      int s = 0, ph = 0, tn = 0;
      auto take = [&](int *idx) -> uint32_t {  // the next ring slot, once its box has landed
        mbar_wait(&full[s], ph);
        const uint32_t p = smem_u32(ring + s * CH_BOX);
        *idx = s;
        if (++s == CH_SLOTS) { s = 0; ph ^= 1; }
        return p;
      };
      // one [128 x 64] A box x one [128 x 64] B box: 4 MMAs of K = 16
      auto mma_box = [&](uint32_t d, uint32_t abox, uint32_t bbox, bool acc) {
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_f16_ss(d, sdesc_sw128(abox + k * 32, 16, 1024), sdesc_sw128(bbox + k * 32, 16, 1024), idesc,
                      (acc || k) ? 1u : 0u);
      };
      const uint32_t aT0 = smem_u32(T0), aTc = smem_u32(Tc), aH = smem_u32(Hb);
      if (a.do_o) {
        for (int kb = 0; kb < a.n_o_kb; ++kb) {
          int sa, sb;
          const uint32_t ab = take(&sa), bb = take(&sb);
          mma_box(tmem + CH_ACC0, ab, bb, kb > 0);
          umma_commit(&empty[sa]);  // the slots are free once these MMAs complete
          umma_commit(&empty[sb]);
        }
        umma_commit(acc_done);
      }
      if (a.do_c) {
        bool t0_waited = false;
        for (int kb = 0; kb < a.nkc; ++kb) {
          uint32_t ab;
          int sa = -1, sb;
          if (kb < a.n_ocat_kb) {
            ab = take(&sa);
          } else {
            if (!t0_waited) {  // o(i) written into T0 by the epilogue
              mbar_wait(t_ready, tn & 1);
              ++tn;
              t0_waited = true;
            }
            ab = aT0 + (kb - a.n_ocat_kb) * CH_BOX;
          }
          const uint32_t bb = take(&sb);
          mma_box(tmem + CH_ACC1, ab, bb, kb > 0);
          if (sa >= 0) umma_commit(&empty[sa]);
          umma_commit(&empty[sb]);
        }
        umma_commit(acc_done);
      }
      if (a.do_c || a.mode == CH_FIRST) {
        if (a.mode == CH_FIRST) {
          mbar_wait(tc_tma, 0);
        } else {
          mbar_wait(t_ready, tn & 1);  // c written into Tc
          ++tn;
        }
        for (int k = 0; k <= a.rd_chunks; ++k) {
          if (k < a.rd_chunks) {  // FFN1(k) -> G[k & 1]
            const int b = k & 1;
            if (k >= 2) mbar_wait(&g_free[b], ((k - 2) >> 1) & 1);
            for (int kb = 0; kb < 2; ++kb) {
              int sb;
              const uint32_t bb = take(&sb);
              mma_box(tmem + CH_G0 + 128 * b, aTc + kb * CH_BOX, bb, kb > 0);
              umma_commit(&empty[sb]);
            }
            umma_commit(&g_done[b]);
          }
          if (k >= 1) {  // FFN2(k - 1): acc0 += H[(k-1) & 1] . Wo^T block
            const int hb = (k - 1) & 1;
            mbar_wait(&h_ready[hb], ((k - 1) >> 1) & 1);
            int sb;
            const uint32_t bb = take(&sb);
            mma_box(tmem + CH_ACC0, aH + hb * CH_BOX, bb, k > 1);
            umma_commit(&h_free[hb]);
            umma_commit(&empty[sb]);
          }
        }
        umma_commit(acc_done);  // q (or z)
      }
      if (a.do_u) {
        mbar_wait(t_ready, tn & 1);  // q written into T0
        ++tn;
        for (int j = 0; j < a.n_u; ++j) {  // U block j -> G[b]; G's FFN phases continue (rd_chunks uses so far)
          const int gi = a.rd_chunks + j, b = gi & 1;
          if (gi >= 2) mbar_wait(&g_free[b], ((gi - 2) >> 1) & 1);
          for (int kb = 0; kb < 2; ++kb) {
            int sb;
            const uint32_t bb = take(&sb);
            mma_box(tmem + CH_G0 + 128 * b, aT0 + kb * CH_BOX, bb, kb > 0);
            umma_commit(&empty[sb]);
          }
          umma_commit(&g_done[b]);
        }
      }
    }
  } else {  // ---------------- epilogue: 8 warps, thread = one row x 64 columns ----------------
    const int q = warp & 3, hg = warp >> 2;
    const int row = q * 32 + lane;
    const int64_t grow = row0 + row;
    const bool ok = grow < a.Nt;
    const uint32_t lanes = (uint32_t)(q * 32) << 16;
    int accn = 0;
    // write 64 values (this thread's half row) as bf16 into an SMEM tile (two SW128 boxes), box = hg
    auto stage_bf16 = [&](uint8_t *T, const float (&y)[64]) {
      uint8_t *box = T + hg * CH_BOX;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4 *>(box + sw128_off(row, c)) =
            make_uint4(pack_bf16(y[8 * c], y[8 * c + 1]), pack_bf16(y[8 * c + 2], y[8 * c + 3]),
                       pack_bf16(y[8 * c + 4], y[8 * c + 5]), pack_bf16(y[8 * c + 6], y[8 * c + 7]));
    };
    auto load64 = [&](uint32_t col, float (&y)[64]) {
      uint32_t r[32];
      tmem_ld32(tmem + lanes + col, r);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; ++e) y[e] = __uint_as_float(r[e]);
      tmem_ld32(tmem + lanes + col + 32, r);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; ++e) y[32 + e] = __uint_as_float(r[e]);
    };
    auto arrive8 = [&](uint64_t *bb) {  // 8 warps -> a count-8 barrier, after generic->async fence
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bb);
    };
    if (a.do_o) {  // o(i): Z (fp32), ocat block i (bf16), T0 (bf16, the A operand of stage c)
      mbar_wait(acc_done, accn & 1);
      ++accn;
      tc_fence_after();
      float y[64];
      load64(CH_ACC0 + 64 * hg, y);
      if (ok) {
        float4 *z4 = reinterpret_cast<float4 *>(a.Z + grow * a.ldz + 64 * hg);
#pragma unroll
        for (int c = 0; c < 16; ++c) z4[c] = make_float4(y[4 * c], y[4 * c + 1], y[4 * c + 2], y[4 * c + 3]);
        uint4 *o4 = reinterpret_cast<uint4 *>(a.ocat + grow * a.ldo + 64 * hg);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          o4[c] = make_uint4(pack_bf16(y[8 * c], y[8 * c + 1]), pack_bf16(y[8 * c + 2], y[8 * c + 3]),
                             pack_bf16(y[8 * c + 4], y[8 * c + 5]), pack_bf16(y[8 * c + 6], y[8 * c + 7]));
      }
      if (a.do_c) {
        stage_bf16(T0, y);
        arrive8(t_ready);
      }
    }
    if (a.do_c) {  // c -> Tc
      mbar_wait(acc_done, accn & 1);
      ++accn;
      tc_fence_after();
      float y[64];
      load64(CH_ACC1 + 64 * hg, y);
      stage_bf16(Tc, y);
      arrive8(t_ready);
    }
    if (a.do_c || a.mode == CH_FIRST) {
      for (int k = 0; k < a.rd_chunks; ++k) {  // SwiGLU of FFN1(k): G[k & 1] -> H[k & 1]
        const int b = k & 1;
        mbar_wait(&g_done[b], (k >> 1) & 1);
        tc_fence_after();
        uint32_t u[32], v[32];
        tmem_ld32(tmem + lanes + CH_G0 + 128 * b + 64 * hg, u);
        tmem_ld32(tmem + lanes + CH_G0 + 128 * b + 64 * hg + 32, v);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&g_free[b]);
        if (k >= 2) mbar_wait(&h_free[b], ((k - 2) >> 1) & 1);  // FFN2(k - 2) has read H[b]
        uint8_t *box = Hb + b * CH_BOX;  // H columns [64 k + 32 hg, + 32) = 16-byte chunks 4 hg .. 4 hg + 3
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float h8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) h8[e] = chain_swiglu(__uint_as_float(u[8 * c + e]), __uint_as_float(v[8 * c + e]));
          *reinterpret_cast<uint4 *>(box + sw128_off(row, 4 * hg + c)) =
              make_uint4(pack_bf16(h8[0], h8[1]), pack_bf16(h8[2], h8[3]), pack_bf16(h8[4], h8[5]), pack_bf16(h8[6], h8[7]));
        }
        arrive8(&h_ready[b]);
      }
      mbar_wait(acc_done, accn & 1);  // q (or z) in acc0
      ++accn;
      tc_fence_after();
      float y[64];
      load64(CH_ACC0 + 64 * hg, y);
      if (a.mode == CH_FIRST) {  // q(1) = LN(.): halves combine (mean, M2) through SMEM
        const float x0 = y[0];
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          const float dd = y[e] - x0;
          s1 += dd;
          s2 = fmaf(dd, dd, s2);
        }
        const float mh = x0 + s1 / 64.f, m2h = fmaxf(s2 - s1 * (s1 / 64.f), 0.f);
        lnx[hg * 128 + row] = make_float2(mh, m2h);
        named_bar_sync(1, 256);
        const float2 o = lnx[(hg ^ 1) * 128 + row];
        const float dm = mh - o.x;
        const float mu = 0.5f * (mh + o.x), var = (m2h + o.y + dm * dm * 32.f) / 128.f;
        const float inv = rsqrtf(var + a.eps);
#pragma unroll
        for (int e = 0; e < 64; ++e) y[e] = fmaf((y[e] - mu) * inv, __ldg(a.g + 64 * hg + e), __ldg(a.b + 64 * hg + e));
      }
      if (a.do_z) {  // z (fp32) out
        if (ok) {
          float4 *z4 = reinterpret_cast<float4 *>(a.zout + grow * CH_D + 64 * hg);
#pragma unroll
          for (int c = 0; c < 16; ++c) z4[c] = make_float4(y[4 * c], y[4 * c + 1], y[4 * c + 2], y[4 * c + 3]);
        }
      } else {
        stage_bf16(T0, y);  // q -> T0 (o(i) in T0 was consumed by stage c, which completed before FFN1)
        arrive8(t_ready);
      }
    }
    if (a.do_u) {
      for (int j = 0; j < a.n_u; ++j) {  // U block j: columns [128 j, + 128) of [N_t x h d]
        const int gi = a.rd_chunks + j, b = gi & 1;
        mbar_wait(&g_done[b], (gi >> 1) & 1);
        tc_fence_after();
        float y[64];
        load64(CH_G0 + 128 * b + 64 * hg, y);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&g_free[b]);
        if (ok) {
          uint4 *u4 = reinterpret_cast<uint4 *>(a.U + grow * a.ldu + 128 * j + 64 * hg);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            u4[c] = make_uint4(pack_bf16(y[8 * c], y[8 * c + 1]), pack_bf16(y[8 * c + 2], y[8 * c + 3]),
                               pack_bf16(y[8 * c + 4], y[8 * c + 5]), pack_bf16(y[8 * c + 6], y[8 * c + 7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc(tmem, 512);
}

}  // namespace tc
}  // namespace stca

namespace stca {

bool tc_chain_supported(int d, int h, int rd) { return d == tc::CH_D && rd % 128 == 0 && (h * d) % 128 == 0; }

cudaError_t tc_chain(const TcChain &c, cudaStream_t st) {
  using namespace tc;
  if (c.Nt <= 0) return cudaSuccess;
  const int d = CH_D, hd = c.h * d;
  CUtensorMap mY, mOc, mWVO, mWC, mW1, mWo, mWQK;
  if (!make_map_bf16(&mOc, c.ocat, c.Nt, (int64_t)(c.M + 1) * d, (int64_t)(c.M + 1) * d, 128)) return cudaErrorInvalidValue;
  mY = mWVO = mWC = mW1 = mWo = mWQK = mOc;  // unused maps: any valid one (never loaded)
  if (c.Y && !make_map_bf16(&mY, c.Y, c.Nt, hd, hd, 128)) return cudaErrorInvalidValue;
  if (c.WVOt && !make_map_bf16(&mWVO, c.WVOt, d, hd, hd, 128)) return cudaErrorInvalidValue;
  if (c.WCt && !make_map_bf16(&mWC, c.WCt, d, (int64_t)c.kc * d, (int64_t)c.kc * d, 128)) return cudaErrorInvalidValue;
  if (c.W1t && !make_map_bf16(&mW1, c.W1t, 2 * c.rd, d, d, 128)) return cudaErrorInvalidValue;
  if (c.Wot && !make_map_bf16(&mWo, c.Wot, d, c.rd, c.rd, 128)) return cudaErrorInvalidValue;
  if (c.WQKt && !make_map_bf16(&mWQK, c.WQKt, hd, d, d, 128)) return cudaErrorInvalidValue;
  ChainArgs a{};
  a.mode = c.mode;
  a.M = c.M;
  a.n_o_kb = hd / 64;
  a.nkc = 2 * c.kc;
  a.n_ocat_kb = 2 * (c.kc - 1);
  a.n_u = hd / 128;
  a.rd_chunks = c.rd / 64;
  a.Nt = (int)c.Nt;
  a.Z = c.Z;
  a.ldz = c.ldz;
  a.ocat = (bf16 *)c.ocat_out;
  a.ldo = (int64_t)(c.M + 1) * d;
  a.U = (bf16 *)c.U;
  a.ldu = hd;
  a.zout = c.zout;
  a.g = c.g;
  a.b = c.b;
  a.eps = c.eps;
  a.do_o = c.mode != CH_FIRST;
  a.do_c = c.mode == CH_MID || (c.mode == CH_LAST && c.zout != nullptr);
  a.do_u = c.mode != CH_LAST;
  a.do_z = c.mode == CH_LAST && c.zout != nullptr;
  cudaError_t e0 = smem_optin((const void *)k_tc_chain, CH_SMEM);
  if (e0 != cudaSuccess) return e0;
  note_launch();
  return launch_pdl(k_tc_chain, dim3((unsigned)((c.Nt + 127) / 128)), dim3(CH_THREADS), (size_t)CH_SMEM, st, mY, mOc,
                    mWVO, mWC, mW1, mWo, mWQK, a);
}

}  // namespace stca
