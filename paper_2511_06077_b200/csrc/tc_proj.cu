// tc_proj.cu -- fused history projection on tcgen05 (sm_100a), SURVEY §2.2 K-A:
//
//   X~(i) = LN(SwiGLUFFN(i)(X)),  i = 1..M,   PAPER.md Eq.(1)-(2)
//
// computed once per request (RLB) from raw X (reading R4) for all M layers in ONE
// launch.  Each CTA owns 128 rows; its X tile is written ONCE into tensor memory and used as the
// TMEM-resident A operand of every layer's first GEMM, and the hidden activation H never leaves
// the SM (TMEM -> registers -> TMEM).  Per layer, the hidden width rd is processed in chunks of 64:
//   GEMM1  G = X . [Wu_c | Wv_c]   tcgen05.mma kind::f16, A = X (TMEM), B = W1 chunk (SMEM), N = 128
//   SwiGLU H_c = u * silu(v)       8 epilogue warps, one row x 32 columns per thread -> bf16 -> TMEM
//   GEMM2  Y += H_c . Wo_c         A = H_c (TMEM), B = Wo chunk (SMEM, MN-major), N = d = 128
// G and H are double-buffered in TMEM (X 64 + Y 128 + H 2x32 + G 2x128 = 512 columns), so the
// epilogue of chunk c overlaps GEMM1 of chunk c+1 and GEMM2 of chunk c-1.  Weights stream through
// a 3-stage TMA ring (48 KB per chunk, L2-resident); with both operands of an SS MMA in SMEM the
// MMAs alone would saturate shared-memory bandwidth, with A in TMEM they read only B (64 B/clk).
// After the last chunk the LayerNorm epilogue (biased variance, eps inside the sqrt) normalises Y
// in registers, stages bf16 X~ rows in SMEM (SW128) and writes them with TMA bulk stores.
//
// Warp roles (352 threads): 0..7 = epilogue (TMEM lane quarter = warp % 4, column half = warp / 4),
// 8 / 9 = TMA producers of the W1 / Wo rings, 10 = TMEM allocator + GEMM1 issuer, 11 = GEMM2 issuer.  The producer and MMA warps have the highest
// warp ids: the SM's warp arbiter prefers them, so the single issuing thread is never starved.
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
bool make_map_bf16_3d(CUtensorMap *m, const void *ptr, int64_t n2, int64_t n1, int64_t n0, int box1);

constexpr int PJ_D = 128;                            // d (row width of X and X~)
constexpr int PJ_ROWS = 128;                         // rows per CTA
constexpr int PJ_NCH = 64;                           // hidden columns per chunk
constexpr int PJ_S1 = 4;                             // W1 ring slots (freed after GEMM1)
constexpr int PJ_SO = 3;                             // Wo ring slots (freed after GEMM2)
constexpr int PJ_W1_BYTES = 2 * PJ_NCH * PJ_D * 2;   // 32 KB: 128 rows (u 64 | v 64) x 128 K, two 64-K boxes
constexpr int PJ_WO_BYTES = PJ_NCH * PJ_D * 2;       // 16 KB: 64 K-rows x 128 N (MN-major), two 64-N boxes
constexpr int PJ_OUT_BYTES = PJ_ROWS * PJ_D * 2;     // 32 KB X~ staging (two 64-column SW128 boxes)
constexpr int PJ_MAXM = 8;                           // layers supported by the fused kernel
constexpr int PJ_GB_BYTES = PJ_MAXM * 2 * PJ_D * 4;  // LayerNorm gamma/beta
constexpr int PJ_RED_BYTES = 2 * 2 * PJ_ROWS * 4;    // row partial sums (mean, variance) x column half
constexpr int PJ_SMEM = 1024 + PJ_S1 * PJ_W1_BYTES + PJ_SO * PJ_WO_BYTES + PJ_OUT_BYTES + PJ_GB_BYTES + PJ_RED_BYTES + 256;
constexpr int PJ_WP1 = 8, PJ_WPO = 9;                // W1 / Wo ring producer warps
constexpr int PJ_WM = 10, PJ_WM2 = 11;               // GEMM1 / GEMM2 issuer warps (WM also owns TMEM)
constexpr int PJ_THREADS = 384;
// TMEM columns
constexpr uint32_t PJ_TY = 0, PJ_TX = 128, PJ_TH = 192, PJ_TG = 256;

struct ProjArgs {
  const bf16 *X;
  int64_t rows;
  const float *g, *b;  // [M x d] LayerNorm affine
  int M, nch;          // layers, chunks per layer (= rd / 64)
  float eps;
  unsigned long long *trace;  // debug (STCA_TRACE): clock64 stamps of CTA 0, else null
};
#define PJ_TR(slot) \
  do {                                                         \
    if (a.trace && blockIdx.x == 0) a.trace[slot] = clock64(); \
  } while (0)

// u * silu(v) = u * v * sigmoid(v),  sigmoid(v) = 0.5 + 0.5 tanh(v / 2): one MUFU op per gate.
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// two gates at once with packed fp32x2 arithmetic (FMUL2 / FFMA2): half the FMA-pipe instructions
__device__ __forceinline__ uint32_t swiglu2(float u0, float v0, float u1, float v1) {
  const uint64_t v2 = f2_pack(v0, v1), half2 = f2_pack(0.5f, 0.5f);
  const uint64_t hv = f2_mul(v2, half2);
  const uint64_t t2 = f2_pack(tanh_approx(f2_lo(hv)), tanh_approx(f2_hi(hv)));
  const uint64_t sg = f2_fma(t2, half2, half2);           // sigmoid(v) = 0.5 tanh(v/2) + 0.5
  const uint64_t uv = f2_mul(f2_pack(u0, u1), v2);
  const uint64_t h2 = f2_mul(uv, sg);
  return pack_bf16(f2_lo(h2), f2_hi(h2));
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    k_tc_project(const __grid_constant__ CUtensorMap mapW1, const __grid_constant__ CUtensorMap mapWo,
                 const __grid_constant__ CUtensorMap mapOut, const ProjArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *sW1 = smem;                                      // W1 ring
  uint8_t *sWo = sW1 + PJ_S1 * PJ_W1_BYTES;                 // Wo ring
  uint8_t *sOut = sWo + PJ_SO * PJ_WO_BYTES;                // X~ staging, [col half][128 rows x 128 B]
  float *sGB = reinterpret_cast<float *>(sOut + PJ_OUT_BYTES);       // [layer][gamma | beta]
  float *sRed = reinterpret_cast<float *>(sOut + PJ_OUT_BYTES + PJ_GB_BYTES);  // [2][col half][row]
  uint64_t *bar = reinterpret_cast<uint64_t *>(sOut + PJ_OUT_BYTES + PJ_GB_BYTES + PJ_RED_BYTES);
  uint64_t *x_full = bar;                  // 8 warp arrivals
  uint64_t *w1_full = bar + 1;             // PJ_S1 (TMA tx)
  uint64_t *w1_empty = w1_full + PJ_S1;    // PJ_S1: GEMM1 of the slot's chunk done in both CTAs
  uint64_t *wo_full = w1_empty + PJ_S1;    // PJ_SO (TMA tx)
  uint64_t *wo_empty = wo_full + PJ_SO;    // PJ_SO: GEMM2 of the slot's chunk done in both CTAs (also frees H)
  uint64_t *g_full = wo_empty + PJ_SO;     // 2: GEMM1 done
  uint64_t *h_full = g_full + 2;           // 2: 8 warp arrivals (H written)
  uint64_t *g_free = h_full + 2;           // 2: 8 warp arrivals (G read into registers)
  uint64_t *y_full = g_free + 2;           // 1: last GEMM2 of a layer done
  uint64_t *y_free = y_full + 1;           // 1: 8 warp arrivals (Y read)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(y_free + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t row0 = (int64_t)blockIdx.x * PJ_ROWS;
  const int total = a.M * a.nch;  // chunks over all layers

  if (warp == PJ_WP1 && lane == 0) {
    tma_prefetch(&mapW1);
    tma_prefetch(&mapWo);
    tma_prefetch(&mapOut);
    mbar_init(x_full, 8);
    for (int s = 0; s < PJ_S1; ++s) {
      mbar_init(&w1_full[s], 1);
      mbar_init(&w1_empty[s], 2);  // both CTAs of the cluster consumed the (multicast) slot
    }
    for (int s = 0; s < PJ_SO; ++s) {
      mbar_init(&wo_full[s], 1);
      mbar_init(&wo_empty[s], 2);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&g_full[b], 1);
      mbar_init(&h_full[b], 8);
      mbar_init(&g_free[b], 8);
    }
    mbar_init(y_full, 1);
    mbar_init(y_free, 8);
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
      uint8_t *ring = w1 ? sW1 : sWo;
      uint64_t *full = w1 ? w1_full : wo_full, *empty = w1 ? w1_empty : wo_empty;
      const CUtensorMap *map = w1 ? &mapW1 : &mapWo;
      int s = 0, ph = 0, row = 0;
      for (int gc = 0; gc < total; ++gc) {
        mbar_wait(&empty[s], ph ^ 1);
        if (w1) PJ_TR(gc * 16 + 7);
        mbar_expect_tx(&full[s], bytes);
        tma_load_2d_mc(ring + s * bytes + crank * (bytes / 2), map, &full[s], 64 * crank, row, 0x3, keep);
        row += rstep;
        if (++s == nslot) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == PJ_WM) {
    if (lane == 0) {  // ---------------- GEMM1 issuer: G[g] = X . W1_c ----------------
      // Two issuing warps: an mbarrier wait right after a commit leaves the tensor pipe idle for
      // ~100 cycles; with GEMM1 and GEMM2 issued from different warps each one's waits are covered
      // by the other's queued MMAs.  Chunk state is kept incrementally (no runtime division here).
      constexpr uint32_t idesc1 = idesc_bf16(128, 2 * PJ_NCH, 0);  // B K-major, N = 128
      const uint32_t aW1 = smem_u32(sW1);
      mbar_wait(x_full, 0);
      int s1 = 0, s1ph = 0, g = 0, gph = 0;
      for (int gc = 0; gc < total; ++gc) {
        if (gc >= 2) mbar_wait(&g_free[g], gph ^ 1);  // the epilogue has read G[g] of chunk gc-2
        mbar_wait(&w1_full[s1], s1ph);
        PJ_TR(gc * 16 + 0);
        tc_fence_after();
        const uint32_t w1 = aW1 + s1 * PJ_W1_BYTES;
#pragma unroll
        for (int k = 0; k < PJ_D / 16; ++k)
          umma_f16_ts(tmem + PJ_TG + g * 128, tmem + PJ_TX + k * 8,
                      sdesc_sw128(w1 + (k >> 2) * (PJ_W1_BYTES / 2) + (k & 3) * 32, 16, 1024), idesc1, k != 0);
        umma_commit(&g_full[g]);
        umma_commit_mc(&w1_empty[s1], 0x3);  // the W1 slot is free again in both CTAs
        PJ_TR(gc * 16 + 1);
        if (++s1 == PJ_S1) { s1 = 0; s1ph ^= 1; }
        g ^= 1;
        if (g == 0) gph ^= 1;
      }
    }
  } else if (warp == PJ_WM2) {
    if (lane == 0) {  // ---------------- GEMM2 issuer: Y += H[g] . Wo_c ----------------
      constexpr uint32_t idesc2 = idesc_bf16(128, PJ_D, 1);  // B MN-major, N = 128
      const uint32_t aWo = smem_u32(sWo);
      int so = 0, soph = 0, g = 0, gph = 0, c = 0, i = 0;
      for (int gc = 0; gc < total; ++gc) {
        mbar_wait(&h_full[g], gph);
        PJ_TR(gc * 16 + 2);
        if (c == 0 && i > 0) mbar_wait(y_free, (i - 1) & 1);  // LN of layer i-1 has read Y
        mbar_wait(&wo_full[so], soph);
        tc_fence_after();
        const uint32_t wo = aWo + so * PJ_WO_BYTES;
#pragma unroll
        for (int k = 0; k < PJ_NCH / 16; ++k)
          umma_f16_ts(tmem + PJ_TY, tmem + PJ_TH + g * 32 + k * 8, sdesc_sw128(wo + k * 2048, PJ_WO_BYTES / 2, 1024),
                      idesc2, (c | k) != 0);
        umma_commit_mc(&wo_empty[so], 0x3);  // frees the Wo slot (and H buffer) in both CTAs
        if (c == a.nch - 1) umma_commit(y_full);
        PJ_TR(gc * 16 + 3);
        if (++so == PJ_SO) { so = 0; soph ^= 1; }
        g ^= 1;
        if (g == 0) gph ^= 1;
        if (++c == a.nch) { c = 0; ++i; }
      }
    }
  } else {  // ---------------- epilogue: 8 warps, row = lane quarter, 64 columns of Y / 32 of H each ----------------
    const int q = warp & 3, hh = warp >> 2;
    const int r = q * 32 + lane;  // row within the tile = TMEM lane
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int64_t grow = row0 + r;
    {  // X row (this thread's 64 columns) -> TMEM as the packed bf16 A operand of GEMM1
      uint32_t w[32];
      const uint4 *src = reinterpret_cast<const uint4 *>(a.X + grow * PJ_D + 64 * hh);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint4 v = grow < a.rows ? src[k] : make_uint4(0, 0, 0, 0);
        w[4 * k] = v.x;
        w[4 * k + 1] = v.y;
        w[4 * k + 2] = v.z;
        w[4 * k + 3] = v.w;
      }
      tmem_st32(tmem + lane_off + PJ_TX + 32 * hh, w);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(x_full);
    }
    for (int i = 0; i < a.M; ++i) {
      for (int c = 0; c < a.nch; ++c) {
        const int gc = i * a.nch + c, g = gc & 1;
        mbar_wait(&g_full[g], (gc >> 1) & 1);
        if (lane == 0 && warp == 0) PJ_TR(gc * 16 + 4);
        tc_fence_after();
        uint32_t u[32], v[32];
        tmem_ld32(tmem + lane_off + PJ_TG + g * 128 + 32 * hh, u);
        tmem_ld32(tmem + lane_off + PJ_TG + g * 128 + 64 + 32 * hh, v);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&g_free[g]);  // G[g] may be overwritten by GEMM1 of chunk gc+2
        if (lane == 0 && warp == 0) PJ_TR(gc * 16 + 5);
        uint32_t h[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          h[j] = swiglu2(__uint_as_float(u[2 * j]), __uint_as_float(v[2 * j]), __uint_as_float(u[2 * j + 1]),
                         __uint_as_float(v[2 * j + 1]));
        if (gc >= 2) mbar_wait(&wo_empty[(gc - 2) % PJ_SO], ((gc - 2) / PJ_SO) & 1);  // GEMM2(gc-2) read H[g]
        if (lane == 0 && warp == 0) PJ_TR(gc * 16 + 6);
        tmem_st16(tmem + lane_off + PJ_TH + g * 32 + 16 * hh, h);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&h_full[g]);
        if (lane == 0) PJ_TR(gc * 16 + 8 + warp);
      }
      // ---- LayerNorm epilogue of layer i ----
      mbar_wait(y_full, i & 1);
      if (lane == 0 && warp == 0) PJ_TR(4096 + i * 4);
      tc_fence_after();
      uint32_t y[64];
      tmem_ld32(tmem + lane_off + PJ_TY + 64 * hh, *reinterpret_cast<uint32_t(*)[32]>(&y[0]));
      tmem_ld32(tmem + lane_off + PJ_TY + 64 * hh + 32, *reinterpret_cast<uint32_t(*)[32]>(&y[32]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(y_free);  // Y may now be overwritten by layer i+1
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int e = 0; e < 64; ++e) s4[e & 3] += __uint_as_float(y[e]);
      sRed[hh * PJ_ROWS + r] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      named_bar_sync(1, 256);
      const float mu = (sRed[r] + sRed[PJ_ROWS + r]) * (1.f / PJ_D);
      float v4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const float dd = __uint_as_float(y[e]) - mu;
        v4[e & 3] = fmaf(dd, dd, v4[e & 3]);
      }
      sRed[2 * PJ_ROWS + hh * PJ_ROWS + r] = (v4[0] + v4[1]) + (v4[2] + v4[3]);
      named_bar_sync(1, 256);
      const float inv = rsqrtf((sRed[2 * PJ_ROWS + r] + sRed[3 * PJ_ROWS + r]) * (1.f / PJ_D) + a.eps);
      const float nmi = -mu * inv;
      const float *gg = sGB + i * 2 * PJ_D + 64 * hh, *bb = gg + PJ_D;
      uint8_t *stage = sOut + hh * (PJ_OUT_BYTES / 2);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 g0 = *reinterpret_cast<const float4 *>(gg + 8 * k);
        const float4 g1 = *reinterpret_cast<const float4 *>(gg + 8 * k + 4);
        const float4 b0 = *reinterpret_cast<const float4 *>(bb + 8 * k);
        const float4 b1 = *reinterpret_cast<const float4 *>(bb + 8 * k + 4);
        const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = fmaf(fmaf(__uint_as_float(y[8 * k + j]), inv, nmi), gv[j], bv[j]);
        *reinterpret_cast<uint4 *>(stage + sw128_off(r, k)) =
            make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
      }
      fence_proxy_async();
      named_bar_sync(1, 256);  // the tile's rows are staged
      if (warp == 0 && lane == 0) {
        tma_store_3d(&mapOut, sOut, 0, (int32_t)row0, i);
        tma_store_3d(&mapOut, sOut + PJ_OUT_BYTES / 2, 64, (int32_t)row0, i);
        bulk_commit();
        bulk_wait_read0();  // staging may be overwritten once the store has read it
      }
      named_bar_sync(1, 256);
      if (lane == 0 && warp == 0) PJ_TR(4096 + i * 4 + 1);
    }
    if (warp == 0 && lane == 0) bulk_wait0();  // all X~ stores of this tile complete
  }
  tc_fence_before();
  cluster_sync_all();  // the peer no longer multicasts into / arrives on this CTA
  if (warp == PJ_WM) tmem_dealloc(tmem, 512);
}

}  // namespace tc

cudaError_t tc_project(const TcProj &p, cudaStream_t st) {
  if (p.rows <= 0) return cudaSuccess;
  if (p.d == tc::PJ_D && p.rd % tc::PJ_NCH == 0 && p.W1cat && p.Wocat && p.gcat && p.bcat &&
      p.out_layer_stride == p.rows * p.d && p.M <= tc::PJ_MAXM) {
    CUtensorMap m1, mo, mout;
    if (!tc::make_map_bf16(&m1, p.W1cat, (int64_t)p.M * 2 * p.rd, p.d, p.d, 2 * tc::PJ_NCH) ||
        !tc::make_map_bf16(&mo, p.Wocat, (int64_t)p.M * p.rd, p.d, p.d, tc::PJ_NCH) ||
        !tc::make_map_bf16_3d(&mout, p.out, p.M, p.rows, p.d, tc::PJ_ROWS))
      return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(tc::k_tc_project, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::PJ_SMEM);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    tc::ProjArgs a{(const bf16 *)p.X, p.rows, p.gcat, p.bcat, p.M, p.rd / tc::PJ_NCH, p.eps, nullptr};
    const char *trace_path = getenv("STCA_TRACE");  // debug only: clock64 stamps of CTA 0
    if (trace_path && cudaMalloc(&a.trace, 8192 * 8) == cudaSuccess) cudaMemsetAsync(a.trace, 0, 8192 * 8, st);
    note_launch();
    const unsigned tiles = (unsigned)((p.rows + tc::PJ_ROWS - 1) / tc::PJ_ROWS);
    tc::k_tc_project<<<(tiles + 1) & ~1u, tc::PJ_THREADS, tc::PJ_SMEM, st>>>(m1, mo, mout, a);  // clusters of 2
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
  const int64_t R = 1 << 18;
  for (int i = 0; i < p.M; ++i) {
    for (int64_t r0 = 0; r0 < p.rows; r0 += R) {
      const int64_t rows = std::min<int64_t>(R, p.rows - r0);
      const bf16 *x = (const bf16 *)p.X + r0 * p.d;
      bf16 *out = (bf16 *)p.out + (int64_t)i * p.out_layer_stride + r0 * p.d;
      cudaError_t e = tc_ffn(x, p.d, rows, p.W1[i], p.Wo[i], p.d, p.rd, p.g[i], p.b[i], p.eps, out, p.d, nullptr, 0, st);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace stca
