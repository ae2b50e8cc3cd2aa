// tc_gemm.cu -- warp-specialised tcgen05 GEMM for sm_100a with fused epilogues.
//
//   C[M x N] = A[M x K] . Bt^T,   A bf16 row-major (lda), Bt = B^T bf16 [N x K] (K-major)
//
// Warps 0-3: epilogue; warp 4: TMA producer (SWIZZLE_128B boxes of 64 K-elements); warp 5: TMEM
// allocator + single-thread tcgen05.mma issuer of the CTA pair (cta_group::2: M = 256 over the two
// CTAs of a cluster, N-slices <= 256, K = 16 per instruction;
// highest warp ids so the arbiter never starves the issuing thread).  Epilogue: one thread per accumulator row (TMEM lane), reading the fp32
// accumulator with tcgen05.ld.  Epilogues:
//   TEPI_STORE  : alpha*acc -> bf16 (Cs) and/or fp32 (Cf)
//   TEPI_SWIGLU : Bt rows chunk-interleaved [u_32c..u_32c+31 | v_32c..v_32c+31]:
//                H[:, 32c+j] = u * silu(v) -> bf16   (Eq.(1))
//   TEPI_LN     : BN == N == d: LayerNorm over the row (biased variance, eps inside sqrt)
//                -> bf16 / fp32                       (Eq.(2)-(3))
//   TEPI_SWIGLU_BWD : the backward of the SwiGLU gate (NEXT-1, hist_bwd.cu) on the recomputed
//                [u | v] chunks of TEPI_SWIGLU's layout: with dH read from global (aux, row-major),
//                da = dH silu(v) -> Cs[:, j], dv = dH u sig(v) (1 + v (1 - sig(v))) -> Cs[:, off2 + j]
// Used for the target-side contractions (U = q W_QK, o = Y W_VO, [o|x_t] W_C, W_Z) and
// the query-side SwiGLUFFN instances.
#include <cudaTypedefs.h>
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <mutex>

#include "launch.h"
#include "tc.h"
#include "tc_ptx.cuh"

namespace stca {
namespace tc {

enum { TEPI_STORE = 0, TEPI_SWIGLU = 1, TEPI_LN = 2, TEPI_SWIGLU_BWD = 3 };

struct EpiArgs {
  bf16 *Cs;
  int64_t ldcs;
  float *Cf;
  int64_t ldcf;
  const float *g, *b;
  float eps;
  const bf16 *aux;  // TEPI_SWIGLU_BWD: dH [M x N/2] bf16, row stride ldaux; dv at column off2 of Cs
  int64_t ldaux, off2;
};

// u * silu(v) = u v sigmoid(v) = a + a tanh(v / 2) with a = u v / 2: one MUFU op per output
__device__ __forceinline__ float swiglu_f(float u, float v) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * v));
  const float a = 0.5f * u * v;
  return fmaf(a, t, a);
}

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int NS = BN < 256 ? BN : 256;  // N per (M = 256, CTA pair) MMA instruction
  static constexpr int A_BYTES = BM * BK * 2;     // 16 KB: this CTA's 128 rows of A
  static constexpr int B_BYTES = BN / 2 * BK * 2;  // this CTA's half of every NS-row block of B^T
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int F_STRIDE = 32 * 4 + 16;    // staged fp32 row of a 32-column output block (bytes)
  static constexpr int H_STRIDE = 32 * 2 + 16;    // staged bf16 row
  static constexpr int STG_BYTES = 128 * F_STRIDE;  // one staged output block per epilogue half (the ring keeps running)
  static constexpr int LNP_BYTES = 2 * BN * 4 + 2 * 128 * 8;  // LayerNorm gamma | beta, half-row statistics
  static constexpr int STAGES_FIT = (227 * 1024 - 2 * STG_BYTES - LNP_BYTES - 1024 - 256) / STAGE;
  static constexpr int STAGES = STAGES_FIT > 6 ? 6 : STAGES_FIT;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : BN <= 256 ? 256 : 512;
  static constexpr int NACC = TMEM_COLS <= 256 ? 2 : 1;  // TMEM accumulators (double-buffered when they fit)
  static constexpr int SMEM = STAGES * STAGE + 2 * STG_BYTES + LNP_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// PERSISTENT: grid = 2 x min(tile pairs, co-resident clusters); cluster c takes 256-row tile pairs
// c, c + clusters, ... (n fastest).  The
// smem ring runs across tiles and the TMEM accumulator is double-buffered, so the epilogue of tile
// i (TMEM -> registers -> padded smem block -> coalesced 16-byte stores) overlaps the MMAs of tile
// i+1 and the loads of tile i+2; per-tile launch / prologue / pipeline-fill costs are paid once
// per SM instead of once per tile (these GEMMs are small: M = N_t = 16384 rows).
constexpr int GEMM_THREADS = 320;  // epilogue warps 0-7, TMA producer 8, MMA issuer 9

template <int BN, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int M, int N,
              int K, float alpha, EpiArgs ea) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *stg = smem + C::STAGES * C::STAGE;
  float *lnp = reinterpret_cast<float *>(stg + 2 * C::STG_BYTES);  // LN: gamma [BN] | beta [BN]
  float2 *lnx = reinterpret_cast<float2 *>(lnp + 2 * BN);           // LN: (mean, M2) of each half row
  uint64_t *full = reinterpret_cast<uint64_t *>(stg + 2 * C::STG_BYTES + C::LNP_BYTES);
  uint64_t *empty = full + C::STAGES;
  uint64_t *acc_full = empty + C::STAGES;   // NACC (MMA commit: accumulator a complete)
  uint64_t *acc_empty = acc_full + 2;       // NACC, leader only (16 epilogue warps of the pair: accumulator a read)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(acc_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // CTA pairs (cta_group::2): a pair computes a 256 x BN tile with M = 256 MMAs issued by the leader
  // (rank 0); CTA r holds A rows [128 r, 128 r + 128) and half of every NS-row block of B^T, so each
  // SM receives 16 KB of A + BN/2 x 64 x 2 bytes of B per 64-deep k-block instead of the whole B —
  // per-SM operand ingest, not L2, is what limits M = 128 tiles at BN >= 256 (a 2-CTA TMA multicast
  // of B measured within 2%: every SM still receives all of B).
  // Tile pairs are numbered n-fastest: the pairs in flight share a few 256-row blocks of A (read
  // from HBM once) and sweep all of B (the weights, L2-resident).
  const int tiles_m = (M + C::BM - 1) / C::BM, tn = N / BN, npairs = (tiles_m + 1) / 2 * tn;
  const int nk = (K + C::BK - 1) / C::BK;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);  // the leader's MMAs have read the slot (commit multicast to both CTAs)
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 16);
    }
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc_pair(tslot, C::NACC * C::TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();  // barrier inits visible cluster-wide before the peer multicasts into this CTA
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t crank = cluster_ctarank();
  pdl_wait();     // the predecessor's outputs (our A) are complete and visible
  pdl_trigger();  // the successor may be scheduled (it waits for us the same way)

  if (warp == 8) {
    if (lane == 0) {  // TMA producer
      int s = 0, ph = 0;
      for (int p = cid; p < npairs; p += ncl) {
        const int m0 = (2 * (p / tn) + (int)crank) * C::BM, n0 = (p % tn) * BN;  // m0 >= M: TMA zero-fills
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t *sa = smem + s * C::STAGE, *sb = sa + C::A_BYTES;
          const uint32_t fb = mapa_shared(&full[s], 0);  // both CTAs' bytes complete on the leader's barrier
          if (crank == 0) mbar_expect_tx(&full[s], 2 * C::STAGE);
          tma_load_2d_pair(sa, &mapA, fb, kb * C::BK, m0, policy_evict_normal());
#pragma unroll
          for (int j = 0; j < BN / C::NS; ++j)  // this CTA's half of each NS-row block of B^T
            tma_load_2d_pair(sb + j * (C::NS / 2) * 128, &mapB, fb, kb * C::BK,
                             n0 + j * C::NS + (int)crank * (C::NS / 2), policy_evict_last());
          if (++s == C::STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0 && crank == 0) {  // MMA issuer (the pair's leader)
      constexpr uint32_t idesc = idesc_bf16(256, C::NS, 0);
      int s = 0, ph = 0, i = 0;
      for (int p = cid; p < npairs; p += ncl, ++i) {
        const int a = i % C::NACC;
        mbar_wait(&acc_empty[a], ((i / C::NACC) & 1) ^ 1);  // the epilogue has read this accumulator
        tc_fence_after();
        const uint32_t acc = tmem + a * C::TMEM_COLS;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * C::STAGE), sb = sa + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k) {
            const uint64_t ad = sdesc_sw128(sa + k * 32, 16, 1024);
#pragma unroll
            for (int j = 0; j < BN / C::NS; ++j) {
              const uint64_t bd = sdesc_sw128(sb + j * (C::NS / 2) * 128 + k * 32, 16, 1024);
              umma_f16_ss_pair(acc + j * C::NS, ad, bd, idesc, (kb | k) != 0);
            }
          }
          umma_commit_pair_mc(&empty[s], 0x3);  // the slot is free again in both CTAs
          if (++s == C::STAGES) { s = 0; ph ^= 1; }
        }
        umma_commit_pair_mc(&acc_full[a], 0x3);  // both CTAs' accumulator halves are complete
      }
    }
  } else {  // epilogue warps 0..7: TMEM lane quarter = warp & 3, column half hg = warp >> 2
    // Each half group (4 warps, 128 threads: all 128 rows, half of the columns) stages a 32-column
    // output block in its own SMEM buffer with padded rows and copies it out with coalesced 16-byte
    // stores (a row per thread written straight to global touches 32 sectors per store).  Two
    // warps per TMEM lane quarter halve the epilogue, which bounds NACC = 1 tiles (BN = 512).
    const int q = warp & 3, hg = warp >> 2, ltid = threadIdx.x & 127;
    const int row = q * 32 + lane;
    uint8_t *hstg = stg + hg * C::STG_BYTES;
    // columns of the accumulator this half group owns (a half group may own none for tiny BN)
    constexpr bool GATE = EPI == TEPI_SWIGLU || EPI == TEPI_SWIGLU_BWD;  // [u 32 | v 32] column blocks
    constexpr int GRAN = GATE ? 64 : 32;
    constexpr bool SPLIT = BN >= 2 * GRAN;
    constexpr int HCOLS = SPLIT ? BN / 2 : BN;
    const int c_lo = SPLIT ? hg * HCOLS : 0;
    const bool active = SPLIT || hg == 0;
    constexpr int OUT_COLS = GATE ? BN / 2 : BN;  // output columns of a tile
    if (EPI == TEPI_LN) {  // gamma/beta from SMEM: global loads in flight stall this warp's tcgen05.ld
      for (int c = threadIdx.x; c < BN; c += 256) {
        lnp[c] = ea.g[c];
        lnp[BN + c] = ea.b[c];
      }
      named_bar_sync(3, 256);
    }
    // TEPI_SWIGLU_BWD: this thread's row of dH for its half group's hidden columns (HCOLS / 2 bf16,
    // contiguous) is loaded one tile AHEAD into registers: eight epilogue warps with one 64-byte load
    // each in flight left the kernel at ~2.5 TB/s (latency-bound), ncu l4_hist_bwd
    constexpr int NBW = EPI == TEPI_SWIGLU_BWD ? HCOLS / 16 : 1;
    uint4 dh_nxt[NBW];
    auto fetch_dh = [&](int pp) {
      if constexpr (EPI == TEPI_SWIGLU_BWD) {
        const int mm = (2 * (pp / tn) + (int)crank) * C::BM, nn = (pp % tn) * BN;
        const int64_t gr = (int64_t)mm + row;
        const bool ok = pp < npairs && gr < M;
        const uint4 *src = reinterpret_cast<const uint4 *>(ea.aux + (ok ? gr : 0) * ea.ldaux + nn / 2 + c_lo / 2);
#pragma unroll
        for (int k = 0; k < NBW; ++k) dh_nxt[k] = ok ? __ldg(src + k) : make_uint4(0, 0, 0, 0);
      }
    };
    fetch_dh(cid);
    int i = 0;
    for (int p = cid; p < npairs; p += ncl, ++i) {
      const int m0 = (2 * (p / tn) + (int)crank) * C::BM, n0 = (p % tn) * BN;
      const int64_t out_n0 = GATE ? n0 / 2 : n0;
      const int a = i % C::NACC;
      mbar_wait(&acc_full[a], (i / C::NACC) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + a * C::TMEM_COLS + ((uint32_t)(q * 32) << 16) + c_lo;
      // stage output block `blk` (32 output columns of the tile, fp32 or bf16 rows), then store it
      auto emit = [&](int blk, const float (&y)[32], bool f32, int64_t coff = 0) {
        const int RS = f32 ? C::F_STRIDE : C::H_STRIDE, ES = f32 ? 4 : 2;
        uint8_t *srow = hstg + row * RS;
        if (f32) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<float4 *>(srow + 16 * k) = make_float4(y[4 * k], y[4 * k + 1], y[4 * k + 2], y[4 * k + 3]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            *reinterpret_cast<uint4 *>(srow + 16 * k) =
                make_uint4(pack_bf16(y[8 * k], y[8 * k + 1]), pack_bf16(y[8 * k + 2], y[8 * k + 3]),
                           pack_bf16(y[8 * k + 4], y[8 * k + 5]), pack_bf16(y[8 * k + 6], y[8 * k + 7]));
        }
        named_bar_sync(1 + hg, 128);
        uint8_t *dst = f32 ? reinterpret_cast<uint8_t *>(ea.Cf) : reinterpret_cast<uint8_t *>(ea.Cs);
        const int64_t ld = f32 ? ea.ldcf : ea.ldcs;
        const int sh = f32 ? 3 : 2;  // log2(16-byte chunks per staged row)
#pragma unroll 4
        for (int c = ltid; c < (128 << sh); c += 128) {
          const int rr = c >> sh, ch = c & ((1 << sh) - 1);
          if ((int64_t)m0 + rr < M)
            *reinterpret_cast<uint4 *>(dst + (((int64_t)m0 + rr) * ld + coff + out_n0 + blk * 32) * ES + ch * 16) =
                *reinterpret_cast<const uint4 *>(hstg + rr * RS + ch * 16);
        }
        named_bar_sync(1 + hg, 128);  // the staging block may be rewritten
      };
      // TMEM blocks are double-buffered in registers: block j+1's tcgen05.ld is in flight while block
      // j is converted and stored (fully unrolled, so the buffer index is static).
      if (EPI == TEPI_STORE) {
        if (active) {
          uint32_t r[2][32];
          tmem_ld32(taddr, r[0]);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < HCOLS; c += 32) {
            const int bi = (c / 32) & 1;
            if (c + 32 < HCOLS) tmem_ld32(taddr + c + 32, r[bi ^ 1]);
            float y[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) y[e] = alpha * __uint_as_float(r[bi][e]);
            if (ea.Cf) emit((c_lo + c) / 32, y, true);
            if (ea.Cs) emit((c_lo + c) / 32, y, false);
            tmem_ld_wait();
          }
        }
      } else if (EPI == TEPI_SWIGLU) {
        if (active) {
          uint32_t u[2][32], v[2][32];
          tmem_ld32(taddr, u[0]);
          tmem_ld32(taddr + 32, v[0]);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < HCOLS; c += 64) {
            const int bi = (c / 64) & 1;
            if (c + 64 < HCOLS) {
              tmem_ld32(taddr + c + 64, u[bi ^ 1]);
              tmem_ld32(taddr + c + 96, v[bi ^ 1]);
            }
            float y[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) y[e] = swiglu_f(__uint_as_float(u[bi][e]), __uint_as_float(v[bi][e]));
            emit((c_lo + c) / 64, y, false);
            tmem_ld_wait();
          }
        }
      } else if (EPI == TEPI_SWIGLU_BWD) {
        uint4 dcur[NBW];
#pragma unroll
        for (int k = 0; k < NBW; ++k) dcur[k] = dh_nxt[k];
        fetch_dh(p + ncl);  // the next tile's dH, in flight during this tile
#pragma unroll
        for (int c = 0; c < HCOLS; c += 64) {
          const int blk = (c_lo + c) / 64;
          uint32_t u[32], v[32];
          tmem_ld32(taddr + c, u);
          tmem_ld32(taddr + c + 32, v);
          float dh[32];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint4 w = dcur[(c / 64) * 4 + k];
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&ww[t]));
              dh[8 * k + 2 * t] = f.x;
              dh[8 * k + 2 * t + 1] = f.y;
            }
          }
          tmem_ld_wait();
          float y[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {  // sig(v) = 1/2 + tanh(v/2)/2 (one MUFU op, as the forward)
            const float vv = __uint_as_float(v[e]);
            float t;
            asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * vv));
            const float sg = fmaf(0.5f, t, 0.5f);
            y[e] = dh[e] * vv * sg;                                                                 // da
            v[e] = __float_as_uint(dh[e] * __uint_as_float(u[e]) * sg * fmaf(vv, 1.f - sg, 1.f));  // dv
          }
          emit(blk, y, false);
#pragma unroll
          for (int e = 0; e < 32; ++e) y[e] = __uint_as_float(v[e]);
          emit(blk, y, false, ea.off2);
        }
      } else if (active) {  // TEPI_LN over BN == d columns
        // one statistics pass over the half row, sums shifted by its first value (no cancellation
        // for rows whose mean is large against their spread); the halves' (mean, M2) combine as
        // mean = (m_0 + m_1)/2, M2 = M2_0 + M2_1 + (m_0 - m_1)^2 n/4 (n = BN, equal halves)
        uint32_t r[2][32];
        tmem_ld32(taddr, r[0]);
        tmem_ld_wait();
        const float x0 = __uint_as_float(r[0][0]);
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int c = 0; c < HCOLS; c += 32) {
          const int bi = (c / 32) & 1;
          if (c + 32 < HCOLS) tmem_ld32(taddr + c + 32, r[bi ^ 1]);
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float d0 = __uint_as_float(r[bi][e]) - x0;
            s1 += d0;
            s2 = fmaf(d0, d0, s2);
          }
          tmem_ld_wait();
        }
        tmem_ld32(taddr, r[0]);  // first block of the output pass, in flight during the exchange
        const float mh = x0 + s1 / HCOLS, m2h = fmaxf(s2 - s1 * (s1 / HCOLS), 0.f);
        float mu, var;
        if (SPLIT) {
          lnx[hg * 128 + row] = make_float2(mh, m2h);
          named_bar_sync(3, 256);
          const float2 o = lnx[(hg ^ 1) * 128 + row];
          const float dm = mh - o.x;
          mu = 0.5f * (mh + o.x);
          var = (m2h + o.y + dm * dm * (0.25f * BN)) / BN;
        } else {
          mu = mh;
          var = m2h / BN;
        }
        const float inv = rsqrtf(var + ea.eps);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < HCOLS; c += 32) {
          const int bi = (c / 32) & 1;
          if (c + 32 < HCOLS) tmem_ld32(taddr + c + 32, r[bi ^ 1]);
          float y[32];
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 g4 = *reinterpret_cast<const float4 *>(lnp + c_lo + c + e);
            const float4 b4 = *reinterpret_cast<const float4 *>(lnp + BN + c_lo + c + e);
            y[e] = fmaf((__uint_as_float(r[bi][e]) - mu) * inv, g4.x, b4.x);
            y[e + 1] = fmaf((__uint_as_float(r[bi][e + 1]) - mu) * inv, g4.y, b4.y);
            y[e + 2] = fmaf((__uint_as_float(r[bi][e + 2]) - mu) * inv, g4.z, b4.z);
            y[e + 3] = fmaf((__uint_as_float(r[bi][e + 3]) - mu) * inv, g4.w, b4.w);
          }
          if (ea.Cf) emit((c_lo + c) / 32, y, true);
          if (ea.Cs) emit((c_lo + c) / 32, y, false);
          tmem_ld_wait();
        }
        if (SPLIT) named_bar_sync(3, 256);  // lnx of this tile consumed before the next tile writes it
      }
      static_assert(OUT_COLS >= 32 || EPI == TEPI_SWIGLU, "32-column output blocks");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(mapa_shared(&acc_empty[a], 0));  // the leader may reuse accumulator a
    }
  }
  tc_fence_before();
  cluster_sync_all();  // the peer no longer multicasts into / arrives on this CTA
  if (warp == 9) tmem_dealloc_pair(tmem, C::NACC * C::TMEM_COLS);
}

// bf16 [n2 x n1 x n0] (n0 innermost, contiguous), box = box1 rows x 64 x 1, SWIZZLE_128B
bool make_map_bf16_3d(CUtensorMap *m, const void *ptr, int64_t n2, int64_t n1, int64_t n0, int box1, int64_t s2 = 0);

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

// bf16 row-major [rows x cols] with leading dimension ld (elements); box = box_rows x 64, SWIZZLE_128B
bool make_map_bf16(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), gdim, gstride, box, estride,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// bf16 [n2 x n1 x n0] (n0 contiguous; dim-2 stride s2 elements, default n1 * n0); box = 64 x box1 x 1
bool make_map_bf16_3d(CUtensorMap *m, const void *ptr, int64_t n2, int64_t n1, int64_t n0, int box1, int64_t s2) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t gdim[3] = {(cuuint64_t)n0, (cuuint64_t)n1, (cuuint64_t)n2};
  cuuint64_t gstride[2] = {(cuuint64_t)(n0 * 2), (cuuint64_t)((s2 ? s2 : n1 * n0) * 2)};
  cuuint32_t box[3] = {64, (cuuint32_t)box1, 1};
  cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(ptr), gdim, gstride, box, estride,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int EPI>
static cudaError_t launch_gemm(const void *A, int64_t lda, const void *Bt, int64_t M, int N, int K, float alpha,
                               const EpiArgs &ea, cudaStream_t st) {
  using C = GemmCfg<BN>;
  CUtensorMap ma, mb;
  if (!make_map_bf16(&ma, A, M, K, lda, 128) || !make_map_bf16(&mb, Bt, N, K, K, C::NS / 2)) return cudaErrorInvalidValue;
  cudaError_t e0 = smem_optin((const void *)k_tc_gemm<BN, EPI>, C::SMEM);
  if (e0 != cudaSuccess) return e0;
  const int mc = cluster_occupancy((const void *)k_tc_gemm<BN, EPI>, GEMM_THREADS, C::SMEM, 2);  // co-resident pairs
  const int64_t npairs = ((M + 127) / 128 + 1) / 2 * (N / BN);
  note_launch();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * std::min<int64_t>(npairs, mc)));
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (launch.h)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_tc_gemm<BN, EPI>, ma, mb, (int)M, N, K, alpha, ea);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace tc

// dispatch on N (N % BN == 0; BN = min(N, 256) for STORE/SWIGLU, BN = N for LN)
static cudaError_t gemm_dispatch(int epi, const void *A, int64_t lda, const void *Bt, int64_t M, int N, int K,
                                 const tc::EpiArgs &ea, cudaStream_t st) {
  using namespace tc;
  if (M <= 0) return cudaSuccess;
  if (K % 64 || N % 32) return cudaErrorInvalidValue;
#define G(BN, E) return launch_gemm<BN, E>(A, lda, Bt, M, N, K, 1.f, ea, st)
  if (epi == TEPI_LN) {
    switch (N) {
      case 64: G(64, TEPI_LN);
      case 128: G(128, TEPI_LN);
      case 256: G(256, TEPI_LN);
      case 512: G(512, TEPI_LN);
      default: return cudaErrorInvalidValue;
    }
  }
  if (epi == TEPI_SWIGLU) {
    if (N % 256 == 0) G(256, TEPI_SWIGLU);
    if (N % 128 == 0) G(128, TEPI_SWIGLU);
    if (N % 64 == 0) G(64, TEPI_SWIGLU);
    return cudaErrorInvalidValue;
  }
  if (epi == TEPI_SWIGLU_BWD) {
    if (N % 256 == 0) G(256, TEPI_SWIGLU_BWD);
    if (N % 128 == 0) G(128, TEPI_SWIGLU_BWD);
    return cudaErrorInvalidValue;
  }
  if (N % 256 == 0) G(256, TEPI_STORE);
  if (N % 128 == 0) G(128, TEPI_STORE);
  if (N % 64 == 0) G(64, TEPI_STORE);
  G(32, TEPI_STORE);
#undef G
}

cudaError_t tc_gemm(const void *A, int64_t lda, const void *Bt, int64_t M, int N, int K, void *Cs, int64_t ldcs,
                    float *Cf, int64_t ldcf, cudaStream_t st) {
  tc::EpiArgs ea{(bf16 *)Cs, ldcs, Cf, ldcf, nullptr, nullptr, 0.f};
  return gemm_dispatch(tc::TEPI_STORE, A, lda, Bt, M, N, K, ea, st);
}

// [da | dv] = SwiGLU gate backward of [u | v] = X W1 (recomputed, W1 in TEPI_SWIGLU's interleaved Bt
// layout [2 rd x d]) given dH [rows x rd]: da -> dag[:, 0:rd], dv -> dag[:, rd:2rd] (bf16, row stride lddag)
cudaError_t tc_swiglu_bwd(const void *X, int64_t ldx, int64_t rows, const void *W1, int d, int rd, const void *dH,
                          int64_t ldh, void *dag, int64_t lddag, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  tc::EpiArgs ea{(bf16 *)dag, lddag, nullptr, 0, nullptr, nullptr, 0.f, (const bf16 *)dH, ldh, rd};
  return gemm_dispatch(tc::TEPI_SWIGLU_BWD, X, ldx, W1, rows, 2 * rd, d, ea, st);
}

// ---- SwiGLUFFN (+LN) over rows, as two tcgen05 GEMMs with H (bf16) in the caller's scratch ----
cudaError_t tc_ffn(const void *in, int64_t ldi, int64_t rows, const void *W1, const void *Wo, int d, int rd,
                   const float *g, const float *b, float eps, void *out_s, int64_t ldo, float *out_f, int64_t ldof,
                   void *H, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (!H) return cudaErrorInvalidValue;
  cudaError_t e;
  tc::EpiArgs e1{(bf16 *)H, rd, nullptr, 0, nullptr, nullptr, 0.f};
  e = gemm_dispatch(tc::TEPI_SWIGLU, in, ldi, W1, rows, 2 * rd, d, e1, st);
  if (e != cudaSuccess) return e;
  tc::EpiArgs e2{(bf16 *)out_s, ldo, out_f, ldof, g, b, eps};
  return gemm_dispatch(g ? tc::TEPI_LN : tc::TEPI_STORE, H, rd, Wo, rows, d, rd, e2, st);
}

}  // namespace stca

// Stage-isolated test hook (not part of include/stca.h): one tcgen05 GEMM with the given
// epilogue (0 store, 1 swiglu, 2 layernorm), so tests can compare it with a torch fp32
// reference of the same op.
extern "C" int stca_debug_tc_gemm(int epi, const void *A, int64_t lda, const void *Bt, int64_t M, int N, int K,
                                  void *Cs, int64_t ldcs, float *Cf, int64_t ldcf, const float *g, const float *b,
                                  float eps, void *stream) {
  stca::tc::EpiArgs ea{(stca::bf16 *)Cs, ldcs, Cf, ldcf, g, b, eps};
  return (int)stca::gemm_dispatch(epi, A, lda, Bt, M, N, K, ea, (cudaStream_t)stream);
}
