// tc_proj.cu -- fused history projection on tcgen05 (sm_100a), SURVEY §2.2 K-A:
//
//   X~(i) = LN(SwiGLUFFN(i)(X)),  i = 1..M,   PAPER.md Eq.(1)-(2)
//
// computed once per request (RLB) from raw X (reading R4) for all layers in
// ONE launch: each CTA keeps its 256-row X tile resident in shared memory for all M
// layers and never materialises the [rows x rd] hidden activation in HBM.  Per layer, the
// hidden width rd is processed in chunks of 32 columns:
//   GEMM1  G = X . [Wu_c | Wv_c]     (two M=128 tiles, N = 64, K = d)   -> TMEM (double-buffered)
//   SwiGLU H_c = u * silu(v)         (epilogue warps, one thread per row) -> bf16, SMEM
//   GEMM2  Y += H_c . Wo_c           (two M=128 tiles, N = d, K = 32)   -> TMEM
// and after the last chunk the LayerNorm epilogue normalises each Y row in registers
// (biased variance, eps inside the sqrt) and stores bf16 X~ rows.  Weights stream
// through a 4-stage TMA ring (24 KB per chunk, shared by both M tiles, L2-resident).
//
// Warp roles (320 threads): 0..7 = SwiGLU / LayerNorm epilogue (M tile = warp / 4, TMEM lane
// quarter = warp % 4), 8 = TMA producer, 9 = TMEM allocator + MMA issuer.  The producer and MMA
// warps get the highest warp ids: the SM's warp arbiter prefers higher ids, so the single
// issuing thread is never starved by the busy epilogue warps sharing its scheduler.
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

constexpr int PJ_D = 128;                      // d (row width of X and X~)
constexpr int PJ_ROWS = 256;                   // rows per CTA (two M = 128 tiles)
constexpr int PJ_NCH = 32;                     // hidden columns per chunk
constexpr int PJ_STAGES = 4;
constexpr int PJ_X_BYTES = PJ_ROWS * PJ_D * 2;             // 64 KB
constexpr int PJ_W1_BYTES = 2 * PJ_NCH * PJ_D * 2;         // 16 KB: 64 rows (u|v) x 128 K
constexpr int PJ_WO_BYTES = PJ_NCH * PJ_D * 2;             // 8 KB: 32 K rows x 128 N (MN-major)
constexpr int PJ_STAGE = PJ_W1_BYTES + PJ_WO_BYTES;        // 24 KB
constexpr int PJ_H_BYTES = 128 * 64 * 2;                   // per M tile: 128 rows x 64 (two chunk halves)
constexpr int PJ_GB_BYTES = 16 * 2 * PJ_D * 4;                // LayerNorm gamma/beta of up to 16 layers
constexpr int PJ_SMEM = 1024 + PJ_X_BYTES + PJ_STAGES * PJ_STAGE + 2 * PJ_H_BYTES + PJ_GB_BYTES + 256;
constexpr int PJ_WP = 8, PJ_WM = 9;                          // producer / MMA warps

struct ProjArgs {
  bf16 *out;                 // layer i at out + i * layer_stride
  int64_t layer_stride;      // elements
  const float *g, *b;        // [M x d] LayerNorm affine
  int64_t rows;
  int M, nch;                // layers, chunks per layer (= rd / 32)
  float eps;
  unsigned long long *trace;  // debug (STCA_TRACE): clock64 stamps of CTA 0, else null
};

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// u * silu(v) = u * v * sigmoid(v),  sigmoid(v) = 0.5 + 0.5 tanh(v / 2)  (one MUFU op)
__device__ __forceinline__ float swiglu(float u, float v) {
  return u * v * fmaf(0.5f, tanh_approx(0.5f * v), 0.5f);
}

__global__ void __launch_bounds__(320, 1)
    k_tc_project(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapW1,
                 const __grid_constant__ CUtensorMap mapWo, const __grid_constant__ CUtensorMap mapOut,
                 const ProjArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *sX = smem;                                   // [tile t][col half][128 rows x 128 B]
  uint8_t *sW = sX + PJ_X_BYTES;                        // stages: [W1 64 rows x 128 K][Wo 2 boxes of 32 x 64]
  uint8_t *sH = sW + PJ_STAGES * PJ_STAGE;              // [tile t][128 rows x 128 B]
  float *sGB = reinterpret_cast<float *>(sH + 2 * PJ_H_BYTES);  // [layer][gamma 128 | beta 128]
  uint64_t *bar = reinterpret_cast<uint64_t *>(sH + 2 * PJ_H_BYTES + PJ_GB_BYTES);
  uint64_t *x_full = bar;
  uint64_t *w_full = bar + 1;
  uint64_t *w_empty = w_full + PJ_STAGES;  // = GEMM2 of that stage's chunk done (frees weights + H half)
  uint64_t *g_full = w_empty + PJ_STAGES;  // 2
  uint64_t *h_full = g_full + 2;           // 2 (count 256)
  uint64_t *h_free = h_full + 2;           // 2
  uint64_t *y_full = h_free + 2;           // 1
  uint64_t *y_free = y_full + 1;           // 1 (count 256)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(y_free + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t row0 = (int64_t)blockIdx.x * PJ_ROWS;
  const int total = a.M * a.nch;  // chunks over all layers

  if (warp == PJ_WP && lane == 0) {
    tma_prefetch(&mapX);
    tma_prefetch(&mapW1);
    tma_prefetch(&mapWo);
    mbar_init(x_full, 1);
    for (int s = 0; s < PJ_STAGES; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&g_full[b], 1);
      mbar_init(&h_full[b], 256);
      mbar_init(&h_free[b], 1);
    }
    mbar_init(y_full, 1);
    mbar_init(y_free, 256);
    fence_mbar_init();
  }
  if (warp == PJ_WM) tmem_alloc(tslot, 512);
  for (int k = threadIdx.x; k < a.M * PJ_D; k += blockDim.x) {
    sGB[(k / PJ_D) * 2 * PJ_D + k % PJ_D] = a.g[k];
    sGB[(k / PJ_D) * 2 * PJ_D + PJ_D + k % PJ_D] = a.b[k];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // TMEM: Y tile t at cols [128 t, 128 t + 128); G buffer g, tile t at 256 + 128 g + 64 t (u 32 | v 32)

  if (warp == PJ_WP) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      const uint64_t keep = policy_evict_last();
      mbar_expect_tx(x_full, PJ_X_BYTES);
      for (int t = 0; t < 2; ++t)
        for (int hc = 0; hc < 2; ++hc)
          tma_load_2d(sX + (t * 2 + hc) * (PJ_X_BYTES / 4), &mapX, x_full, hc * 64, (int32_t)(row0 + t * 128));
      for (int gc = 0; gc < total; ++gc) {
        const int s = gc % PJ_STAGES, i = gc / a.nch, c = gc % a.nch;
        mbar_wait(&w_empty[s], ((gc / PJ_STAGES) & 1) ^ 1);
        uint8_t *w1 = sW + s * PJ_STAGE, *wo = w1 + PJ_W1_BYTES;
        mbar_expect_tx(&w_full[s], PJ_STAGE);
        const int32_t r1 = i * 2 * a.nch * PJ_NCH + c * 2 * PJ_NCH;  // W1^T rows of this chunk (u 32 | v 32)
        tma_load_2d_hint(w1, &mapW1, &w_full[s], 0, r1, keep);
        tma_load_2d_hint(w1 + PJ_W1_BYTES / 2, &mapW1, &w_full[s], 64, r1, keep);
        const int32_t ro = i * a.nch * PJ_NCH + c * PJ_NCH;           // Wo rows (K) of this chunk
        tma_load_2d_hint(wo, &mapWo, &w_full[s], 0, ro, keep);
        tma_load_2d_hint(wo + PJ_WO_BYTES / 2, &mapWo, &w_full[s], 64, ro, keep);
      }
    }
  } else if (warp == PJ_WM) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc1 = idesc_bf16(128, 2 * PJ_NCH, 0);  // G = X W1c : B K-major, N = 64
      constexpr uint32_t idesc2 = idesc_bf16(128, PJ_D, 1);        // Y += H Wo_c : B MN-major, N = 128
      const uint32_t aX = smem_u32(sX), aW = smem_u32(sW), aH = smem_u32(sH);
      mbar_wait(x_full, 0);
      auto gemm2 = [&](int gc) {
        const int s = gc % PJ_STAGES, g = gc & 1, i = gc / a.nch, c = gc % a.nch;
        mbar_wait(&h_full[g], (gc >> 1) & 1);
        if (a.trace && blockIdx.x == 0) a.trace[gc * 16 + 2] = clock64();
        if (c == 0 && i > 0) mbar_wait(y_free, (i - 1) & 1);  // LN of layer i-1 has read Y
        tc_fence_after();
        const uint32_t wo = aW + s * PJ_STAGE + PJ_W1_BYTES;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
#pragma unroll
          for (int k = 0; k < PJ_NCH / 16; ++k) {
            const uint64_t ad = sdesc_sw128(aH + t * PJ_H_BYTES + g * 64 + k * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(wo + k * 2048, PJ_WO_BYTES / 2, 1024);
            umma_f16_ss(tmem + t * 128, ad, bd, idesc2, (c | k) != 0);
          }
        }
        if (a.trace && blockIdx.x == 0) a.trace[gc * 16 + 3] = clock64();
        umma_commit(&w_empty[s]);
        if (c == a.nch - 1) umma_commit(y_full);
      };
      for (int gc = 0; gc < total; ++gc) {
        const int s = gc % PJ_STAGES, g = gc & 1;
        mbar_wait(&w_full[s], (gc / PJ_STAGES) & 1);
        if (a.trace && blockIdx.x == 0) a.trace[gc * 16 + 0] = clock64();
        // G buffer g was released by the epilogue of chunk gc-2 (waited on in gemm2(gc-2))
        tc_fence_after();
        const uint32_t w1 = aW + s * PJ_STAGE;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
#pragma unroll
          for (int k = 0; k < PJ_D / 16; ++k) {
            const uint64_t ad = sdesc_sw128(aX + (t * 2 + (k >> 2)) * (PJ_X_BYTES / 4) + (k & 3) * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(w1 + (k >> 2) * (PJ_W1_BYTES / 2) + (k & 3) * 32, 16, 1024);
            umma_f16_ss(tmem + 256 + g * 128 + t * 64, ad, bd, idesc1, k != 0);
          }
        }
        umma_commit(&g_full[g]);
        if (a.trace && blockIdx.x == 0) a.trace[gc * 16 + 1] = clock64();
        if (gc >= 1) gemm2(gc - 1);
      }
      gemm2(total - 1);
    }
  } else {  // ---------------- SwiGLU + LayerNorm epilogue (256 threads) ----------------
    const int t = warp >> 2, q = warp & 3;
    const int r = q * 32 + lane;  // row within the M tile = TMEM lane
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint8_t *hrow = sH + t * PJ_H_BYTES;
    for (int i = 0; i < a.M; ++i) {
      for (int c = 0; c < a.nch; ++c) {
        const int gc = i * a.nch + c, g = gc & 1;
        mbar_wait(&g_full[g], (gc >> 1) & 1);
        if (a.trace && blockIdx.x == 0 && lane == 0 && warp == 0) a.trace[gc * 16 + 4] = clock64();
        tc_fence_after();
        uint32_t u[32], v[32];
        tmem_ld32(tmem + lane_off + 256 + g * 128 + t * 64, u);
        tmem_ld32(tmem + lane_off + 256 + g * 128 + t * 64 + 32, v);
        tmem_ld_wait();
        if (a.trace && blockIdx.x == 0 && lane == 0 && warp == 0) a.trace[gc * 16 + 5] = clock64();
        if (gc >= 2) mbar_wait(&w_empty[(gc - 2) % PJ_STAGES], ((gc - 2) / PJ_STAGES) & 1);  // GEMM2(gc-2) read H half g
        if (a.trace && blockIdx.x == 0 && lane == 0 && warp == 0) a.trace[gc * 16 + 6] = clock64();
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // 4 x 16 B = this chunk's 32 hidden values of row r
          uint32_t w[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int e = 8 * k + 2 * j;
            w[j] = pack_bf16(swiglu(__uint_as_float(u[e]), __uint_as_float(v[e])),
                             swiglu(__uint_as_float(u[e + 1]), __uint_as_float(v[e + 1])));
          }
          *reinterpret_cast<uint4 *>(hrow + sw128_off(r, g * 4 + k)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(&h_full[g]);
        if (a.trace && blockIdx.x == 0 && lane == 0) a.trace[gc * 16 + 8 + warp] = clock64();
      }
      // LayerNorm epilogue of layer i
      mbar_wait(y_full, i & 1);
      if (a.trace && blockIdx.x == 0 && lane == 0 && warp == 0) a.trace[4096 + i * 4 + 0] = clock64();
      tc_fence_after();
      uint32_t y[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t (&rr)[32] = *reinterpret_cast<uint32_t(*)[32]>(&y[32 * c]);
        tmem_ld32(tmem + lane_off + t * 128 + 32 * c, rr);
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(y_free);  // Y may now be overwritten by layer i+1
      if (a.trace && blockIdx.x == 0 && lane == 0 && warp == 0) a.trace[4096 + i * 4 + 1] = clock64();
      float s4[4] = {0.f, 0.f, 0.f, 0.f};  // independent partial sums (short dependency chains)
#pragma unroll
      for (int e = 0; e < PJ_D; ++e) s4[e & 3] += __uint_as_float(y[e]);
      const float mu = ((s4[0] + s4[1]) + (s4[2] + s4[3])) * (1.f / PJ_D);
      float v4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int e = 0; e < PJ_D; ++e) {
        const float dd = __uint_as_float(y[e]) - mu;
        v4[e & 3] = fmaf(dd, dd, v4[e & 3]);
      }
      const float inv = rsqrtf(((v4[0] + v4[1]) + (v4[2] + v4[3])) * (1.f / PJ_D) + a.eps);
      const float nmi = -mu * inv;
      const float *gg = sGB + i * 2 * PJ_D, *bb = gg + PJ_D;  // smem broadcast reads
      // X~ rows leave through the (now idle) H buffer of this M tile as a 128 x 64 SW128 staging tile,
      // written to HBM by one TMA bulk store per 64-column half (coalesced, clipped at the layer end).
      uint8_t *stage = sH + t * PJ_H_BYTES;
#pragma unroll
      for (int hc = 0; hc < 2; ++hc) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int e0 = hc * 64 + 8 * k;
          const float4 g0 = *reinterpret_cast<const float4 *>(gg + e0);
          const float4 g1 = *reinterpret_cast<const float4 *>(gg + e0 + 4);
          const float4 b0 = *reinterpret_cast<const float4 *>(bb + e0);
          const float4 b1 = *reinterpret_cast<const float4 *>(bb + e0 + 4);
          const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
          const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
          float o[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] = fmaf(fmaf(__uint_as_float(y[e0 + j]), inv, nmi), gv[j], bv[j]);
          *reinterpret_cast<uint4 *>(stage + sw128_off(r, k)) =
              make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
        }
        fence_proxy_async();
        named_bar_sync(1 + t, 128);  // the 128 rows of this tile are staged
        if (q == 0 && lane == 0) {
          tma_store_3d(&mapOut, stage, hc * 64, (int32_t)(row0 + t * 128), i);
          bulk_commit();
          bulk_wait_read0();  // staging may be overwritten once the store has read it
        }
        named_bar_sync(1 + t, 128);
      }
    }
    if (q == 0 && lane == 0) bulk_wait0();  // all X~ stores of this tile complete
  }
  tc_fence_before();
  __syncthreads();
  if (warp == PJ_WM) tmem_dealloc(tmem, 512);
}

}  // namespace tc

cudaError_t tc_project(const TcProj &p, cudaStream_t st) {
  if (p.rows <= 0) return cudaSuccess;
  if (p.d == tc::PJ_D && p.rd % 64 == 0 && p.W1cat && p.Wocat && p.gcat && p.bcat) {
    CUtensorMap mx, m1, mo, mout;
    if (!tc::make_map_bf16(&mx, p.X, p.rows, p.d, p.d, 128) ||
        !tc::make_map_bf16(&m1, p.W1cat, (int64_t)p.M * 2 * p.rd, p.d, p.d, 2 * tc::PJ_NCH) ||
        !tc::make_map_bf16(&mo, p.Wocat, (int64_t)p.M * p.rd, p.d, p.d, tc::PJ_NCH) ||
        p.out_layer_stride != p.rows * p.d || !tc::make_map_bf16_3d(&mout, p.out, p.M, p.rows, p.d, 128))
      return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(tc::k_tc_project, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::PJ_SMEM);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    tc::ProjArgs a{(bf16 *)p.out, p.out_layer_stride, p.gcat, p.bcat, p.rows, p.M, p.rd / tc::PJ_NCH, p.eps,
                   nullptr};
    const char *trace_path = getenv("STCA_TRACE");  // debug only: clock64 stamps of CTA 0
    if (trace_path && cudaMalloc(&a.trace, 8192 * 8) == cudaSuccess) cudaMemsetAsync(a.trace, 0, 8192 * 8, st);
    note_launch();
    tc::k_tc_project<<<(unsigned)((p.rows + tc::PJ_ROWS - 1) / tc::PJ_ROWS), 320, tc::PJ_SMEM, st>>>(mx, m1, mo, mout, a);
    if (a.trace) {
      unsigned long long h[8192];
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
