// tc_proj.cu -- fused history projection on tcgen05 (sm_100a), SURVEY §2.2 K-A:
//
//   X~(i) = LN(SwiGLUFFN(i)(X)),  i = 1..M,   PAPER.md Eq.(1)-(2)
//
// computed once per request (RLB) from raw X (reading R4) for all M layers in ONE
// persistent launch (one 2-CTA cluster per SM pair walks 128-row tile pairs).  A CTA's X tile is
// written into tensor memory and used as the TMEM-resident A operand of every layer's first GEMM;
// the hidden activation H never leaves the SM (TMEM -> registers -> TMEM).  Per layer, the hidden
// width rd is processed in chunks of 64:
//   GEMM1  G = X . [Wu_c | Wv_c]   tcgen05.mma kind::f16, A = X (TMEM), B = W1 chunk (SMEM), N = 128
//   SwiGLU H_c = u * silu(v)       two groups of 4 epilogue warps take alternate chunks -> bf16 -> TMEM
//   GEMM2  Y += H_c . Wo_c         A = H_c (TMEM), B = Wo chunk (SMEM, MN-major), N = d = 128
// G and H are double-buffered in TMEM (Y 128 + X 64 + H 2x32 + G 2x128 = 512 columns), so the
// epilogue of chunk c overlaps GEMM1 of chunk c+1 and GEMM2 of chunk c-1.  Weights stream through
// TMA rings (W1 3 x 32 KB, Wo 3 x 16 KB; each CTA of the pair fetches half a slot and multicasts it,
// so weights leave L2 once per pair).  After a layer's last chunk a LayerNorm group (biased
// variance, eps inside the sqrt) releases Y after three TMEM loads (half in registers, half parked
// in SMEM), normalises, stages bf16 X~ rows in SMEM (SW128) and a spare lane writes them with TMA.
//
// Warp roles (512 threads): 0..7 = SwiGLU (TMEM lane quarter = warp % 4, group = warp / 4),
// 8..11 = LayerNorm + next-tile X, 12 / 13 = TMA producers of the W1 / Wo rings (13 lane 16: X~
// stores), 14 = TMEM allocator + GEMM1 issuer, 15 = GEMM2 issuer.  The producer and MMA warps have
// the highest warp ids: the SM's warp arbiter prefers them, so the single issuing thread is never
// starved.  Design notes from measurement (tools/mma_bench, tools/swiglu_bench, STCA_TRACE):
// every tcgen05.commit costs the tensor pipe ~45 cycles (one per GEMM here); a single SwiGLU group
// needs ~1100 cycles per chunk, two alternating groups ~620; global loads issued by any warp hold up
// other warps' tcgen05.ld/st, so the next tile's X arrives by TMA.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "launch.h"
#include "tc.h"
#include "tc_ptx.cuh"

namespace stca {
namespace tc {

bool make_map_bf16(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);
bool make_map_bf16_3d(CUtensorMap *m, const void *ptr, int64_t n2, int64_t n1, int64_t n0, int box1, int64_t s2);

constexpr int PJ_D = 128;                            // d (row width of X and X~)
constexpr int PJ_ROWS = 128;                         // rows per CTA
constexpr int PJ_NCH = 64;                           // hidden columns per chunk
constexpr int PJ_S1 = 3;                             // W1 ring slots (freed after GEMM1)
constexpr int PJ_SO = 3;                             // Wo ring slots (freed after GEMM2)
constexpr int PJ_W1_BYTES = 2 * PJ_NCH * PJ_D * 2;   // 32 KB: 128 rows (u 64 | v 64) x 128 K, two 64-K boxes
constexpr int PJ_WO_BYTES = PJ_NCH * PJ_D * 2;       // 16 KB: 64 K-rows x 128 N (MN-major), two 64-N boxes
constexpr int PJ_OUT_BYTES = PJ_ROWS * PJ_D * 2;     // 32 KB X~ staging (two 64-column SW128 boxes)
constexpr int PJ_MAXM = 8;                           // layers supported by the fused kernel
constexpr int PJ_GB_BYTES = PJ_MAXM * 2 * PJ_D * 4;  // LayerNorm gamma/beta
constexpr int PJ_YS_STRIDE = 64 * 4 + 16;           // fp32 Y columns [64, 128) parked in SMEM, padded rows
constexpr int PJ_YS_BYTES = PJ_ROWS * PJ_YS_STRIDE;
constexpr int PJ_SMEM =
    1024 + PJ_S1 * PJ_W1_BYTES + PJ_SO * PJ_WO_BYTES + PJ_OUT_BYTES + PJ_YS_BYTES + PJ_GB_BYTES + 256;
constexpr int PJ_WLN = 8;                            // warps 8..11: LayerNorm + X group
constexpr int PJ_WP1 = 12, PJ_WPO = 13;              // W1 / Wo ring producer warps
constexpr int PJ_WM = 14, PJ_WM2 = 15;               // GEMM1 / GEMM2 issuer warps (WM also owns TMEM)
constexpr int PJ_THREADS = 512;
// TMEM columns
constexpr uint32_t PJ_TY = 0, PJ_TX = 128, PJ_TH = 192, PJ_TG = 256;

struct ProjArgs {
  const bf16 *X;
  int64_t rows;
  const float *g, *b;  // [M x d] LayerNorm affine
  int M, nch;          // layers, chunks per layer (= rd / 64)
  int npairs;          // 128-row tile pairs (one per cluster iteration)
  float eps;
  unsigned long long *trace;  // debug (STCA_TRACE): clock64 stamps of CTA 0's first tile, else null
};
#define PJ_TRC(gc, k)                                                               \
  do {                                                                              \
    if (a.trace && blockIdx.x == 0 && (gc) < 256) a.trace[(gc) * 16 + (k)] = clock64(); \
  } while (0)
#define PJ_TRL(li, k)                                                                 \
  do {                                                                                \
    if (a.trace && blockIdx.x == 0 && (li) < 16) a.trace[4096 + (li) * 8 + (k)] = clock64(); \
  } while (0)

// u * silu(v) = u * v * sigmoid(v),  sigmoid(v) = 0.5 + 0.5 tanh(v / 2): one MUFU op per gate.
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// two gates at once with packed fp32x2 arithmetic (FMUL2 / FFMA2): half the FMA-pipe instructions.
// u v sigmoid(v) = a + a tanh(v/2) with a = u (v/2): two MUFU ops and three packed FMA-pipe ops.
__device__ __forceinline__ uint32_t swiglu2(float u0, float v0, float u1, float v1) {
  const uint64_t hv = f2_mul(f2_pack(v0, v1), f2_pack(0.5f, 0.5f));  // v / 2
  const uint64_t t2 = f2_pack(tanh_approx(f2_lo(hv)), tanh_approx(f2_hi(hv)));
  const uint64_t a2 = f2_mul(f2_pack(u0, u1), hv);                   // u v / 2
  const uint64_t h2 = f2_fma(a2, t2, a2);
  return pack_bf16(f2_lo(h2), f2_hi(h2));
}

// this thread's 64 columns of X row `grow` (zero past the end) as packed bf16 pairs
__device__ __forceinline__ void load_x_row(const ProjArgs &a, int64_t grow, int hh, uint4 (&x)[8]) {
  const uint4 *src = reinterpret_cast<const uint4 *>(a.X + grow * PJ_D + 64 * hh);
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = grow < a.rows ? __ldg(src + k) : make_uint4(0, 0, 0, 0);
}
__device__ __forceinline__ void store_x_tmem(uint32_t taddr, const uint4 (&x)[8]) {
  uint32_t w[32];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    w[4 * k] = x[k].x;
    w[4 * k + 1] = x[k].y;
    w[4 * k + 2] = x[k].z;
    w[4 * k + 3] = x[k].w;
  }
  tmem_st32(taddr, w);
}

// Persistent: each cluster walks tile pairs cid, cid + nclusters, ...; CTA rank r of the pair owns
// tile 2 * pair + r.  The weight rings, G/H double buffers and the Y / X handshakes run on global
// chunk / layer counters across tiles.
//
// Epilogue: two SwiGLU groups of 4 warps (one warp per TMEM lane quarter, one thread per row) take
// alternate chunks (group = chunk parity = G/H buffer), so one group's TMEM-load latency hides under
// the other's tanh work; a single group cannot reach the MMA rate (~1100 cycles per chunk alone).
// A third group of 4 warps does each layer's LayerNorm and writes the next tile's X into TMEM, so
// neither ever stalls the SwiGLU groups.  The X~ TMA stores are issued by a spare lane of the Wo
// producer warp.  16 warps -> at most 128 registers per thread.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1)
    k_tc_project(const __grid_constant__ CUtensorMap mapW1, const __grid_constant__ CUtensorMap mapWo,
                 const __grid_constant__ CUtensorMap mapOut, const __grid_constant__ CUtensorMap mapX,
                 const ProjArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *sW1 = smem;                                      // W1 ring
  uint8_t *sWo = sW1 + PJ_S1 * PJ_W1_BYTES;                 // Wo ring
  uint8_t *sOut = sWo + PJ_SO * PJ_WO_BYTES;                // X~ staging, [col half][128 rows x 128 B]
  uint8_t *sYs = sOut + PJ_OUT_BYTES;                       // Y columns [64, 128), fp32, one padded row per thread
  float *sGB = reinterpret_cast<float *>(sYs + PJ_YS_BYTES);         // [layer][gamma | beta]
  uint64_t *bar = reinterpret_cast<uint64_t *>(sYs + PJ_YS_BYTES + PJ_GB_BYTES);
  uint64_t *x_full = bar;                  // 1: 4 warp arrivals (X tile in TMEM), one phase per tile
  uint64_t *w1_full = bar + 1;             // PJ_S1 (TMA tx)
  uint64_t *w1_empty = w1_full + PJ_S1;    // PJ_S1: GEMM1 of the slot's chunk done in both CTAs (epilogue arrival)
  uint64_t *wo_full = w1_empty + PJ_S1;    // PJ_SO (TMA tx)
  uint64_t *wo_empty = wo_full + PJ_SO;    // PJ_SO: GEMM2 of the slot's chunk done in both CTAs (also frees H)
  // 4: GEMM1 of chunk gc done in both CTAs (multicast commits), barrier gc & 3.  Four, not one per
  // G buffer: a group that skips chunks must never wait on a barrier two phases ahead of its state
  uint64_t *g_full = wo_empty + PJ_SO;
  uint64_t *h_full = g_full + 4;           // 2: 4 warp arrivals (H written)
  uint64_t *g_free = h_full + 2;           // 2: 4 warp arrivals (G read into registers)
  uint64_t *y_full = g_free + 2;           // 1: a layer's last GEMM2 done (Y complete)
  uint64_t *y_free = y_full + 1;           // 1: 4 warp arrivals (Y read by the LN group)
  uint64_t *st_full = y_free + 1;          // 1: 4 warp arrivals (X~ rows staged)
  uint64_t *st_free = st_full + 1;         // 1: the store lane (staging read by the TMA store)
  uint64_t *x_free = st_free + 1;          // 1: a tile's last GEMM1 done (X may be replaced)
  uint64_t *xs_full = x_free + 1;          // 1: the next tile's X landed in SMEM (TMA tx)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(xs_full + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int ntile = (a.npairs - cid + ncl - 1) / ncl;  // tiles this CTA processes
  const int per_tile = a.M * a.nch;
  const int total = ntile * per_tile;  // chunks over all tiles and layers

  if (warp == PJ_WP1 && lane == 0) {
    tma_prefetch(&mapW1);
    tma_prefetch(&mapWo);
    tma_prefetch(&mapOut);
    tma_prefetch(&mapX);
    mbar_init(x_full, 4);
    for (int s = 0; s < PJ_S1; ++s) {
      mbar_init(&w1_full[s], 1);
      mbar_init(&w1_empty[s], 1);  // this CTA's epilogue saw GEMM1 done in both CTAs
    }
    for (int s = 0; s < PJ_SO; ++s) {
      mbar_init(&wo_full[s], 1);
      mbar_init(&wo_empty[s], 2);
    }
    for (int b = 0; b < 4; ++b) mbar_init(&g_full[b], 2);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&h_full[b], 4);
      mbar_init(&g_free[b], 4);
    }
    mbar_init(y_full, 1);
    mbar_init(y_free, 4);
    mbar_init(st_full, 4);
    mbar_init(st_free, 1);
    mbar_init(x_free, 1);
    mbar_init(xs_full, 1);
    fence_mbar_init();
  }
  if (warp == PJ_WM) tmem_alloc(tslot, 512);
  for (int k = threadIdx.x; k < a.M * PJ_D; k += blockDim.x) {
    sGB[(k / PJ_D) * 2 * PJ_D + k % PJ_D] = a.g[k];
    sGB[(k / PJ_D) * 2 * PJ_D + PJ_D + k % PJ_D] = a.b[k];
  }
  tc_fence_before();
  cluster_sync_all();  // barrier inits visible cluster-wide before the peer multicasts into this CTA
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t crank = cluster_ctarank();

  if (warp == PJ_WP1 || warp == PJ_WPO) {
    if (lane == 0) {  // ---------------- TMA producers (W1 ring / Wo ring) ----------------
      const uint64_t keep = policy_evict_last();
      // each CTA fetches half of every slot (one 64-wide box) for BOTH CTAs of the cluster, so every
      // weight byte leaves L2 once per CTA pair; incremental counters (no runtime division: it would
      // queue on the MUFU pipe, which the SwiGLU epilogue keeps saturated)
      const bool w1 = warp == PJ_WP1;
      const int nslot = w1 ? PJ_S1 : PJ_SO, bytes = w1 ? PJ_W1_BYTES : PJ_WO_BYTES, rstep = w1 ? 2 * PJ_NCH : PJ_NCH;
      const int rend = per_tile * rstep;  // weight rows of all layers: wrap at every tile
      uint8_t *ring = w1 ? sW1 : sWo;
      uint64_t *full = w1 ? w1_full : wo_full, *empty = w1 ? w1_empty : wo_empty;
      const CUtensorMap *map = w1 ? &mapW1 : &mapWo;
      int s = 0, ph = 0, row = 0;
      for (int gc = 0; gc < total; ++gc) {
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], bytes);
        tma_load_2d_mc(ring + s * bytes + crank * (bytes / 2), map, &full[s], 64 * crank, row, 0x3, keep);
        row += rstep;
        if (row == rend) row = 0;
        if (++s == nslot) { s = 0; ph ^= 1; }
      }
    } else if (warp == PJ_WPO && lane == 16) {  // ---------------- X~ store lane ----------------
      int li = 0;
      for (int t = 0; t < ntile; ++t) {
        const int32_t row0 = (2 * (cid + t * ncl) + (int)crank) * PJ_ROWS;
        for (int i = 0; i < a.M; ++i, ++li) {
          mbar_wait(st_full, li & 1);
          tma_store_3d(&mapOut, sOut, 0, row0, i);
          tma_store_3d(&mapOut, sOut + PJ_OUT_BYTES / 2, 64, row0, i);
          bulk_commit();
          bulk_wait_read0();  // the staging buffer has been read
          mbar_arrive(st_free);
        }
      }
      bulk_wait0();  // all X~ stores of this CTA complete
    }
  } else if (warp == PJ_WM) {
    if (lane == 0) {  // ---------------- GEMM1 issuer: G[g] = X . W1_c ----------------
      // Two issuing warps: an mbarrier wait right after a commit leaves the tensor pipe idle for
      // ~100 cycles; with GEMM1 and GEMM2 issued from different warps each one's waits are covered
      // by the other's queued MMAs.  Chunk state is kept incrementally (no runtime division here).
      constexpr uint32_t idesc1 = idesc_bf16(128, 2 * PJ_NCH, 0);  // B K-major, N = 128
      const uint32_t aW1 = smem_u32(sW1);
      int s1 = 0, s1ph = 0, g = 0, gph = 0, c = 0, t = 0;
      for (int gc = 0; gc < total; ++gc) {
        if (c == 0) mbar_wait(x_full, t & 1);  // this tile's X is in TMEM
        if (gc >= 2) mbar_wait(&g_free[g], gph ^ 1);  // the epilogue has read G[g] of chunk gc-2
        mbar_wait(&w1_full[s1], s1ph);
        PJ_TRC(gc, 0);
        tc_fence_after();
        const uint32_t w1 = aW1 + s1 * PJ_W1_BYTES;
#pragma unroll
        for (int k = 0; k < PJ_D / 16; ++k)
          umma_f16_ts(tmem + PJ_TG + g * 128, tmem + PJ_TX + k * 8,
                      sdesc_sw128(w1 + (k >> 2) * (PJ_W1_BYTES / 2) + (k & 3) * 32, 16, 1024), idesc1, k != 0);
        // ONE commit per GEMM: every tcgen05.commit costs the tensor pipe ~45 cycles
        // (tools/mma_bench).  The epilogue, which waits on g_full anyway, frees the W1 slot.
        umma_commit_mc(&g_full[gc & 3], 0x3);
        if (c == per_tile - 1) umma_commit(x_free);  // one extra commit per tile
        PJ_TRC(gc, 1);
        if (++s1 == PJ_S1) { s1 = 0; s1ph ^= 1; }
        g ^= 1;
        if (g == 0) gph ^= 1;
        if (++c == per_tile) { c = 0; ++t; }
      }
    }
  } else if (warp == PJ_WM2) {
    if (lane == 0) {  // ---------------- GEMM2 issuer: Y += H[g] . Wo_c ----------------
      constexpr uint32_t idesc2 = idesc_bf16(128, PJ_D, 1);  // B MN-major, N = 128
      const uint32_t aWo = smem_u32(sWo);
      int so = 0, soph = 0, g = 0, gph = 0, c = 0, li = 0;
      for (int gc = 0; gc < total; ++gc) {
        mbar_wait(&h_full[g], gph);
        PJ_TRC(gc, 2);
        if (c == 0 && li > 0) mbar_wait(y_free, (li - 1) & 1);  // LN of the previous layer has read Y
        mbar_wait(&wo_full[so], soph);
        tc_fence_after();
        const uint32_t wo = aWo + so * PJ_WO_BYTES;
#pragma unroll
        for (int k = 0; k < PJ_NCH / 16; ++k)
          umma_f16_ts(tmem + PJ_TY, tmem + PJ_TH + g * 32 + k * 8, sdesc_sw128(wo + k * 2048, PJ_WO_BYTES / 2, 1024),
                      idesc2, (c | k) != 0);
        umma_commit_mc(&wo_empty[so], 0x3);  // frees the Wo slot and H buffer
        if (c == a.nch - 1) umma_commit(y_full);  // Y complete (one extra commit per layer)
        PJ_TRC(gc, 3);
        if (++so == PJ_SO) { so = 0; soph ^= 1; }
        g ^= 1;
        if (g == 0) gph ^= 1;
        if (++c == a.nch) { c = 0; ++li; }
      }
    }
  } else if (warp < PJ_WLN) {  // ---------------- SwiGLU: 2 groups x 4 warps, thread = one row ----------------
    const int q = warp & 3, grp = warp >> 2;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    for (int gc = grp; gc < total; gc += 2) {
      const int g = grp;  // = gc & 1
      if (lane == 0 && q == 0) PJ_TRC(gc, 7);
      mbar_wait(&g_full[gc & 3], (gc >> 2) & 1);
      if (lane == 0 && q == 0) {
        mbar_arrive(&w1_empty[gc % PJ_S1]);  // GEMM1(gc) no longer reads its W1 slot
        PJ_TRC(gc, 4);
      }
      tc_fence_after();
      uint32_t h[32];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t u[32], v[32];
        tmem_ld32(tmem + lane_off + PJ_TG + g * 128 + 32 * half, u);
        tmem_ld32(tmem + lane_off + PJ_TG + g * 128 + 64 + 32 * half, v);
        tmem_ld_wait();
        if (half == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&g_free[g]);  // G[g] may be overwritten by GEMM1 of chunk gc+2
        }
#pragma unroll
        for (int j = 0; j < 16; ++j)
          h[16 * half + j] = swiglu2(__uint_as_float(u[2 * j]), __uint_as_float(v[2 * j]),
                                     __uint_as_float(u[2 * j + 1]), __uint_as_float(v[2 * j + 1]));
      }
      if (lane == 0 && q == 0) PJ_TRC(gc, 5);
      if (gc >= 2) mbar_wait(&wo_empty[(gc - 2) % PJ_SO], ((gc - 2) / PJ_SO) & 1);  // GEMM2(gc-2) read H[g]
      if (lane == 0 && q == 0) PJ_TRC(gc, 6);
      tmem_st32(tmem + lane_off + PJ_TH + g * 32, h);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&h_full[g]);
      if (lane == 0) PJ_TRC(gc, 8 + warp);
    }
  } else if (warp < PJ_WLN + 4) {  // ---------------- LayerNorm + X group: 4 warps, thread = one row ----------------
    const int q = warp & 3;
    const int r = q * 32 + lane;  // row within the tile = TMEM lane
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t tX = tmem + lane_off + PJ_TX, tY = tmem + lane_off + PJ_TY;
    const int64_t rstride = (int64_t)2 * ncl * PJ_ROWS;  // rows between this CTA's consecutive tiles
    int64_t grow = (int64_t)(2 * cid + crank) * PJ_ROWS + r;  // this thread's row of the current tile
    {
      uint4 x0[8], x1[8];  // a row of X: columns [0, 64) and [64, 128)
      load_x_row(a, grow, 0, x0);  // first tile's X
      load_x_row(a, grow, 1, x1);
      store_x_tmem(tX, x0);
      store_x_tmem(tX + 32, x1);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(x_full);
    int li = 0;
    for (int t = 0; t < ntile; ++t, grow += rstride) {
      for (int i = 0; i < a.M; ++i, ++li) {
        const bool next_x = i == a.M - 1 && t + 1 < ntile;
        if (i == (a.M > 1 ? a.M - 2 : 0) && t + 1 < ntile && q == 0 && lane == 0) {
          // warm L2 with the next tile's X a layer ahead: its TMA load below then hits L2
          const int32_t nrow0 = (int32_t)((grow - r) + rstride);
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(&mapX), "r"(0), "r"(nrow0)
                       : "memory");
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(&mapX), "r"(64), "r"(nrow0)
                       : "memory");
        }
        uint8_t *ys = sYs + r * PJ_YS_STRIDE;  // this thread's padded SMEM row (Y columns [64, 128))
        if (next_x) {
          // the next tile's X tile: TMA -> the (idle) Y-parking SMEM area while this layer's chunks
          // run, then -> TMEM once the tile's last GEMM1 is done.  Plain global loads here were
          // measured to hold up the SwiGLU groups' tcgen05.ld/st for ~2000 cycles (same queue).
          fence_proxy_async();     // this group's earlier reads of the area precede the async write
          named_bar_sync(2, 128);  // (all 4 warps of the group)
          if (q == 0 && lane == 0) {
            const int32_t nrow0 = (int32_t)((grow - r) + rstride);
            mbar_expect_tx(xs_full, PJ_ROWS * PJ_D * 2);
            tma_load_2d(sYs, &mapX, xs_full, 0, nrow0);
            tma_load_2d(sYs + PJ_ROWS * 128, &mapX, xs_full, 64, nrow0);
          }
          if (q == 0 && lane == 0) PJ_TRL(li, 7);
          mbar_wait(xs_full, t & 1);
          if (q == 0 && lane == 0) PJ_TRL(li, 4);
          mbar_wait(x_free, t & 1);
          if (q == 0 && lane == 0) PJ_TRL(li, 5);
          tc_fence_after();
          uint4 x0[8], x1[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            x0[k] = *reinterpret_cast<const uint4 *>(sYs + sw128_off(r, k));
            x1[k] = *reinterpret_cast<const uint4 *>(sYs + PJ_ROWS * 128 + sw128_off(r, k));
          }
          store_x_tmem(tX, x0);
          store_x_tmem(tX + 32, x1);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(x_full);
          if (q == 0 && lane == 0) PJ_TRL(li, 6);
          named_bar_sync(2, 128);  // every row of X read before the area is reused for Y below
        }
        mbar_wait(y_full, li & 1);
        tc_fence_after();
        if (lane == 0 && q == 0) PJ_TRL(li, 0);
        // Release Y fast (the next layer's first GEMM2 waits for it): columns [0, 64) stay in
        // registers, columns [64, 128) are parked in SMEM (this thread's own padded row), then
        // two-pass mean / biased variance (reading R: eps inside the sqrt) and the affine map.
        {  // columns [64, 128) -> SMEM first, so at most 64 registers hold Y at any time
          uint32_t ta[32], tb[32];
          tmem_ld32(tY + 64, ta);
          tmem_ld32(tY + 96, tb);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint4 *>(ys + 16 * k) = make_uint4(ta[4 * k], ta[4 * k + 1], ta[4 * k + 2], ta[4 * k + 3]);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint4 *>(ys + 128 + 16 * k) = make_uint4(tb[4 * k], tb[4 * k + 1], tb[4 * k + 2], tb[4 * k + 3]);
        }
        uint32_t ya[32], yb[32];  // columns [0, 32), [32, 64)
#define YV(e) ((e) < 32 ? ya[(e) & 31] : yb[(e) & 31])
#define Y2(e) f2_pack(__uint_as_float(YV(2 * (e))), __uint_as_float(YV(2 * (e) + 1)))  // packed fp32x2 pair
        tmem_ld32(tY, ya);
        tmem_ld32(tY + 32, yb);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(y_free);  // Y may now be overwritten by the next layer
        if (lane == 0 && q == 0) PJ_TRL(li, 3);
        const uint4 *ys4 = reinterpret_cast<const uint4 *>(ys);
#define YS2(k, h) (h ? (uint64_t)ys4[k].w << 32 | ys4[k].z : (uint64_t)ys4[k].y << 32 | ys4[k].x)  // SMEM pair
        uint64_t s2[2] = {0ull, 0ull};
#pragma unroll
        for (int e = 0; e < 32; ++e) s2[e & 1] = f2_add(s2[e & 1], Y2(e));
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const uint4 v = ys4[k];
          s2[0] = f2_add(s2[0], (uint64_t)v.y << 32 | v.x);
          s2[1] = f2_add(s2[1], (uint64_t)v.w << 32 | v.z);
        }
        const uint64_t st = f2_add(s2[0], s2[1]);
        const float mu = (f2_lo(st) + f2_hi(st)) * (1.f / PJ_D);
        const uint64_t nmu2 = f2_pack(-mu, -mu);
        uint64_t v2[2] = {0ull, 0ull};
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const uint64_t dd = f2_add(Y2(e), nmu2);
          v2[e & 1] = f2_fma(dd, dd, v2[e & 1]);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const uint4 v = ys4[k];
          const uint64_t d0 = f2_add((uint64_t)v.y << 32 | v.x, nmu2), d1 = f2_add((uint64_t)v.w << 32 | v.z, nmu2);
          v2[0] = f2_fma(d0, d0, v2[0]);
          v2[1] = f2_fma(d1, d1, v2[1]);
        }
        const uint64_t vt = f2_add(v2[0], v2[1]);
        const float inv = rsqrtf((f2_lo(vt) + f2_hi(vt)) * (1.f / PJ_D) + a.eps);
        const uint64_t inv2 = f2_pack(inv, inv), nmi2 = f2_pack(-mu * inv, -mu * inv);
        if (li > 0) mbar_wait(st_free, (li - 1) & 1);  // the previous layer's X~ store has read the staging
        if (lane == 0 && q == 0) PJ_TRL(li, 2);
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {  // column half: registers, then SMEM (bounded unrolling: 128-register cap)
          const uint4 *gg = reinterpret_cast<const uint4 *>(sGB + i * 2 * PJ_D + 64 * hb);
          const uint4 *bb = gg + PJ_D / 4;
          uint8_t *stage = sOut + hb * (PJ_OUT_BYTES / 2);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            uint32_t o[4];
            asm volatile("" ::: "memory");  // keep the gamma / beta loads next to their use
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint4 gq = gg[2 * k + j], bq = bb[2 * k + j];
              uint64_t p0, p1;
              if (hb == 0) {
                p0 = Y2(4 * k + 2 * j);
                p1 = Y2(4 * k + 2 * j + 1);
              } else {
                p0 = YS2(2 * k + j, 0);
                p1 = YS2(2 * k + j, 1);
              }
              const uint64_t z0 = f2_fma(f2_fma(p0, inv2, nmi2), (uint64_t)gq.y << 32 | gq.x, (uint64_t)bq.y << 32 | bq.x);
              const uint64_t z1 = f2_fma(f2_fma(p1, inv2, nmi2), (uint64_t)gq.w << 32 | gq.z, (uint64_t)bq.w << 32 | bq.z);
              o[2 * j] = pack_bf16(f2_lo(z0), f2_hi(z0));
              o[2 * j + 1] = pack_bf16(f2_lo(z1), f2_hi(z1));
            }
            *reinterpret_cast<uint4 *>(stage + sw128_off(r, k)) = make_uint4(o[0], o[1], o[2], o[3]);
          }
        }
#undef YS2
#undef YV
#undef Y2
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(st_full);  // the store lane writes the tile's rows once all 4 warps staged
        if (lane == 0 && q == 0) PJ_TRL(li, 1);
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // the peer no longer multicasts into / arrives on this CTA
  if (warp == PJ_WM) tmem_dealloc(tmem, 512);
}

}  // namespace tc

cudaError_t tc_project(const TcProj &p, cudaStream_t st) {
  if (p.rows <= 0) return cudaSuccess;
  if (p.d == tc::PJ_D && p.rd % (2 * tc::PJ_NCH) == 0 && p.rd >= 4 * tc::PJ_NCH &&  // an even number >= 4 of chunks per layer
      p.W1cat && p.Wocat && p.gcat && p.bcat &&
      p.out_layer_stride >= p.rows * p.d && p.out_layer_stride % 8 == 0 && p.M <= tc::PJ_MAXM) {
    CUtensorMap m1, mo, mout, mx;
    if (!tc::make_map_bf16(&m1, p.W1cat, (int64_t)p.M * 2 * p.rd, p.d, p.d, 2 * tc::PJ_NCH) ||
        !tc::make_map_bf16(&mo, p.Wocat, (int64_t)p.M * p.rd, p.d, p.d, tc::PJ_NCH) ||
        !tc::make_map_bf16_3d(&mout, p.out, p.M, p.rows, p.d, tc::PJ_ROWS, p.out_layer_stride) ||
        !tc::make_map_bf16(&mx, p.X, p.rows, p.d, p.d, tc::PJ_ROWS))
      return cudaErrorInvalidValue;
    auto kern = tc::k_tc_project;
    cudaError_t e0 = smem_optin((const void *)kern, tc::PJ_SMEM);
    if (e0 != cudaSuccess) return e0;
    // persistent grid: as many 2-CTA clusters as can be co-resident (1 CTA per SM)
    const int mc = cluster_occupancy((const void *)kern, tc::PJ_THREADS, tc::PJ_SMEM, 2);
    const int64_t tiles = (p.rows + tc::PJ_ROWS - 1) / tc::PJ_ROWS;
    const int npairs = (int)((tiles + 1) / 2);
    tc::ProjArgs a{(const bf16 *)p.X, p.rows, p.gcat, p.bcat, p.M, p.rd / tc::PJ_NCH, npairs, p.eps, nullptr};
    const char *trace_path = getenv("STCA_TRACE");  // debug only: clock64 stamps of CTA 0
    if (trace_path && cudaMalloc(&a.trace, 8192 * 8) == cudaSuccess) cudaMemsetAsync(a.trace, 0, 8192 * 8, st);
    note_launch();
    kern<<<2 * std::min(npairs, mc), tc::PJ_THREADS, tc::PJ_SMEM, st>>>(m1, mo, mout, mx, a);  // clusters of 2
    if (a.trace) {
      static unsigned long long h[8192];
      cudaMemcpyAsync(h, a.trace, sizeof h, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      cudaFree(a.trace);
      if (FILE *f = fopen(trace_path, "wb")) {
        fwrite(h, sizeof h, 1, f);
        fclose(f);
      }
    }
    return cudaGetLastError();
  }
  // other widths: per layer, two tcgen05 GEMMs (SwiGLU epilogue -> H bf16, then W_o + LN epilogue)
  const int64_t R = p.H_rows;
  if (!p.H || R <= 0) return cudaErrorInvalidValue;
  for (int i = 0; i < p.M; ++i) {
    for (int64_t r0 = 0; r0 < p.rows; r0 += R) {
      const int64_t rows = std::min<int64_t>(R, p.rows - r0);
      const bf16 *x = (const bf16 *)p.X + r0 * p.d;
      bf16 *out = (bf16 *)p.out + (int64_t)i * p.out_layer_stride + r0 * p.d;
      cudaError_t e = tc_ffn(x, p.d, rows, p.W1[i], p.Wo[i], p.d, p.rd, p.g[i], p.b[i], p.eps, out, p.d, nullptr, 0, p.H, st);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace stca
