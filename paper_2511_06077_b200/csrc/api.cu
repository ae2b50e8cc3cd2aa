// api.cu -- the C ABI of include/stca.h: validation, host planning (exact integer
// work), device memory ownership and the orchestration of the
// STCA forward under RLB (§3.1-3.2).  Kernels live in kernels_*.cu / tc_*.cu.
#include <cuda.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/stca.h"
#include "launch.h"
#include "tc.h"

#define STCA_H2D_PIECES 8  // pieces of a pipelined host-input projection
// default split-K chunk cap: a 10k history runs as 2 chunks (measured: 4096 -> 3 chunks cost the serve
// forward ~9% more in partial traffic and merge; no split at all balances the persistent grid worse)
#define STCA_DEFAULT_CHUNK_KEYS 8192

using stca::bf16;

#include <atomic>
static std::atomic<int64_t> g_launches{0};
namespace stca {
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace stca

namespace {

// Working-buffer provider of a handle (stca_alloc_fn, include/stca.h): the caller's (e.g. PyTorch's
// caching allocator) or the CUDA stream-ordered pool.  Never synchronises the device.
struct Alloc {
  stca_alloc_fn fa = nullptr;
  stca_free_fn ff = nullptr;
  void *ctx = nullptr;
  int dev = 0;
  cudaError_t get(void **p, size_t bytes, cudaStream_t st) const {
    if (fa) {
      *p = fa(ctx, bytes, dev, (void *)st);
      return *p ? cudaSuccess : cudaErrorMemoryAllocation;
    }
    return cudaMallocAsync(p, bytes, st);
  }
  void put(void *p, cudaStream_t st) const {
    if (!p) return;
    if (ff)
      ff(ctx, p, dev, (void *)st);
    else
      cudaFreeAsync(p, st);
  }
};

// A grow-only device buffer; the old block is released in stream order on the stream that grows it
// (work already enqueued there may still read it).
struct DevBuf {
  void *p = nullptr;
  size_t cap = 0;
  const Alloc *al = nullptr;
  cudaError_t ensure(size_t bytes, cudaStream_t st) {
    if (bytes <= cap) return cudaSuccess;
    al->put(p, st);
    p = nullptr;
    cap = 0;
    size_t want = bytes + bytes / 8 + 256;
    cudaError_t e = al->get(&p, want, st);
    if (e == cudaSuccess)
      cap = want;
    else
      p = nullptr;
    return e;
  }
  void release() {  // the device is idle (stca_destroy)
    if (p && al) al->put(p, 0);
    p = nullptr;
    cap = 0;
  }
  template <typename T> T *as() const { return reinterpret_cast<T *>(p); }
};

struct HostPinned {
  void *p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    size_t want = bytes + bytes / 8 + 256;
    cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocMapped | cudaHostAllocPortable);  // read by kernels too
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

// Pinned staging ring for host-side plans (work lists, gather segments): slot k is reused (and
// possibly regrown) only after the event recorded behind its last H2D copy, so a call never waits
// for the device unless STAGING_SLOTS calls are still in flight.
constexpr int STAGING_SLOTS = 8;
struct StagingRing {
  HostPinned buf[STAGING_SLOTS];
  cudaEvent_t ev[STAGING_SLOTS] = {};
  int next = 0;
  void release() {
    for (int k = 0; k < STAGING_SLOTS; ++k) {
      buf[k].release();
      if (ev[k]) cudaEventDestroy(ev[k]);
      ev[k] = nullptr;
    }
  }
};

// Per-phase event regions (stca_profile)
struct ProfRegion {
  int phase;
  cudaEvent_t a, b;
};

}  // namespace

// rows per block of the history backward (hist_bwd.cu): 2^18 rows keep its weight-gradient GEMMs
// (K = rows) out of the small split-K shapes; scratch ~1.2 GB at d = 128, r = 4
#define STCA_BWD_ROWS (1 << 18)

struct LayerW {
  void *W1h = nullptr, *Woh = nullptr;  // history FFN: [d x 2rd] interleaved (u_j, v_j), [rd x d]
  float *gh = nullptr, *bh = nullptr;
  void *W1cat = nullptr;                // history FFN [Wu | Wv] [d x 2rd] row-major (the backward's GEMMs)
  void *W1q = nullptr, *Woq = nullptr;  // query FFN
  float *gq = nullptr, *bq = nullptr;   // layer 1 only
  void *WQK = nullptr;                  // [d x h d], scaled by log2(e)/sqrt(d_h)
  void *WVO = nullptr;                  // [h d x d]
  void *WC = nullptr;                   // [(i) d x d], rows permuted to the Ocat layout [x_t|o1|..]
  stca::TcWeights tc;                   // tcgen05 repacks (bf16 path)
};

struct stca_handle {
  stca_config cfg{};
  std::string err;
  bool sticky = false;
  bool bf16 = true;
  int es = 2;  // storage element size
  std::vector<void *> allocs;
  LayerW L[STCA_MAX_LAYERS];
  void *W1z = nullptr, *Woz = nullptr, *WZ = nullptr;
  stca::TcWeights tcz;
  stca::TcProjWeights tcp;  // all layers' history FFN/LN, concatenated for the fused projection
  // projection state
  int64_t B = -1;
  std::vector<int64_t> start, len, coff;  // start'_b (input rows), L'_b, compacted offsets [B+1]
  std::vector<int64_t> own0, olen;         // split-history: first owned key and owned key count (else 0, L'_b)
  int64_t T2 = 0;
  Alloc al;
  DevBuf xt_cache;  // M x [T2 x d] storage
  DevBuf xin[2], xgather, seg, proj_h, proj_y;  // xin: double-buffered host-input staging
  // forward scratch
  DevBuf xtin, ocat, q, c, hbuf, ybuf32, U, Y, part, partg, plan, zout, Zout;  // plan: [items | merge items | CTA lists]
  StagingRing stage;
  // session cache (stca_session_open / stca_project_history_session): X~ rows per user across calls
  struct SessEntry {
    int64_t gen, len, off;
  };
  bool sess_on = false;
  int64_t sess_cap = 0, sess_head = 0;
  std::map<int64_t, SessEntry> sess;      // user -> entry
  std::map<int64_t, int64_t> sess_pos;    // cache row offset -> user (ordered, for eviction by overlap)
  void *blas = nullptr;  // cuBLAS handle of the backward (created on first use)
  DevBuf bwd_scratch;
  // stca_backward: fp32 copies of the target-side weights (user orientation; bf16 path, d = 128 only),
  // the forward's per-layer U and Y (save_act), the target-side scratch, dX~ of one layer, unrequested gradients
  std::map<std::string, float *> w32;
  bool save_act = false;
  // split-history over peer memory (stca_split_peer_export / stca_split_peer_attach)
  void *peer_buf = nullptr;  // this rank's exchange buffer (cudaMalloc): [4 KB: ready[64], device UUID at 1024 | slot 0 | slot 1]
  int64_t peer_cap = 0;      // bytes per slot
  bool peer_on = false;
  void **peer_tab = nullptr;  // device: [slot 0 of rank g][slot 1 of rank g][ready flags of g], G each
  uint64_t epoch = 0;         // one per layer of every split forward (identical on all ranks)
  std::vector<uint8_t *> peer_bases;  // host copy of the G buffers' addresses
  uint8_t peer_uuid[16] = {};         // this device's UUID (also at byte 1024 of the exported buffer)
  // NEXT-3 (i): the standard attention form (stca_set_attention_form): per layer W_Q and [W_K | W_V]
  // zero-padded to d columns per head, W_O rows per head at the V block, in the tcgen05 layout
  int attn_form = 0;
  stca::TcWeights std_q[STCA_MAX_LAYERS], std_kv[STCA_MAX_LAYERS];
  DevBuf kvbuf;  // [T' x h d]: per history row and head [K^r | V^r | 0]
  DevBuf act, sbwd_scratch, dxt_buf, gsink, dxsink;
  // stca_debug_capture (stage-isolated tests): copy U and Y of one layer during the next forward
  int cap_layer = 0;
  void *cap_U = nullptr, *cap_Y = nullptr;
  // stca_profile
  bool prof = false, prof_target = false;
  int reps_attn = 1, reps_proj = 1;  // STCA_PROF_TWICE_*
  std::vector<ProfRegion> prof_open;  // recorded, not yet read
  std::vector<cudaEvent_t> prof_pool;
  int64_t chunk_cap = STCA_DEFAULT_CHUNK_KEYS;
  // pipelined host-input projection: copy stream + one event per piece
  cudaStream_t copy_st = nullptr;
  cudaEvent_t ev_xin_free[2] = {}, ev[STCA_H2D_PIECES] = {};
  cudaEvent_t ev_xtin_free = nullptr, ev_xt_in = nullptr;  // host x_t upload on the copy stream
  int xin_k = 0;  // staging buffer of the next host-input projection
};

static DevBuf *const *all_bufs(stca_handle *h, int *n) {
  static thread_local DevBuf *v[32];
  DevBuf *list[] = {&h->act, &h->sbwd_scratch, &h->dxt_buf, &h->gsink, &h->dxsink, &h->kvbuf,
                    &h->xt_cache, &h->xin[0], &h->xin[1], &h->bwd_scratch, &h->xgather, &h->seg,    &h->proj_h, &h->proj_y, &h->xtin,
                    &h->ocat,     &h->q,    &h->c,       &h->hbuf,   &h->ybuf32, &h->U,      &h->Y,
                    &h->part,     &h->partg, &h->plan,   &h->zout,   &h->Zout};
  *n = (int)(sizeof list / sizeof list[0]);
  for (int i = 0; i < *n; ++i) v[i] = list[i];
  return v;
}

// ---- stca_profile: event regions on the launching stream ----
static cudaEvent_t prof_begin(stca_handle *h, cudaStream_t st) {
  if (!h->prof) return nullptr;
  cudaEvent_t e = nullptr;
  if (!h->prof_pool.empty()) {
    e = h->prof_pool.back();
    h->prof_pool.pop_back();
  } else if (cudaEventCreate(&e) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  cudaEventRecord(e, st);
  return e;
}
static void prof_end(stca_handle *h, int phase, cudaEvent_t a, cudaStream_t st) {
  if (!a) return;
  cudaEvent_t b = nullptr;
  if (!h->prof_pool.empty()) {
    b = h->prof_pool.back();
    h->prof_pool.pop_back();
  } else if (cudaEventCreate(&b) != cudaSuccess) {
    cudaGetLastError();
    h->prof_pool.push_back(a);
    return;
  }
  cudaEventRecord(b, st);
  h->prof_open.push_back({phase, a, b});
}

static thread_local std::string g_create_error;  // message of the last failed stca_create on this thread

static stca_status fail(stca_handle *h, stca_status s, const char *fmt, ...) __attribute__((format(printf, 3, 4)));
static stca_status fail(stca_handle *h, stca_status s, const char *fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    h->err = buf;
    if (s == STCA_ERR_CUDA) h->sticky = true;
  }
  return s;
}

#define CU(expr)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      if (e_ == cudaErrorMemoryAllocation) {                                                       \
        cudaGetLastError();                                                                        \
        return fail(h, STCA_ERR_OOM, "%s: %s", #expr, cudaGetErrorString(e_));                     \
      }                                                                                            \
      return fail(h, STCA_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e_)); \
    }                                                                                              \
  } while (0)

// ===========================================================================
// host planning (exact integer work)
// ===========================================================================
extern "C" {

int32_t stca_abi_version(void) { return STCA_ABI_VERSION; }

int64_t stca_kernel_launches(void) { return g_launches.load(); }

const char *stca_status_string(int32_t s) {
  switch (s) {
    case STCA_OK: return "STCA_OK";
    case STCA_ERR_INVALID_ARG: return "STCA_ERR_INVALID_ARG";
    case STCA_ERR_SHAPE: return "STCA_ERR_SHAPE";
    case STCA_ERR_OFFSETS: return "STCA_ERR_OFFSETS";
    case STCA_ERR_EMPTY_HISTORY: return "STCA_ERR_EMPTY_HISTORY";
    case STCA_ERR_UNSUPPORTED: return "STCA_ERR_UNSUPPORTED";
    case STCA_ERR_STATE: return "STCA_ERR_STATE";
    case STCA_ERR_OOM: return "STCA_ERR_OOM";
    case STCA_ERR_CUDA: return "STCA_ERR_CUDA";
    case STCA_ERR_COMM: return "STCA_ERR_COMM";
    default: return "STCA_ERR_UNKNOWN";
  }
}

static stca_status check_offsets(const int64_t *off, int64_t B, int64_t rows, bool nonempty, int64_t *bad) {
  *bad = -1;
  if (B < 0) return STCA_ERR_INVALID_ARG;
  if (!off) return STCA_ERR_INVALID_ARG;
  if (off[0] != 0) return STCA_ERR_OFFSETS;
  for (int64_t b = 0; b < B; ++b)
    if (off[b + 1] < off[b]) {
      *bad = b;
      return STCA_ERR_OFFSETS;
    }
  if (off[B] != rows) return STCA_ERR_OFFSETS;
  if (nonempty)
    for (int64_t b = 0; b < B; ++b)
      if (off[b + 1] == off[b]) {
        *bad = b;
        return STCA_ERR_EMPTY_HISTORY;
      }
  return STCA_OK;
}

stca_status stca_validate_offsets(const int64_t *hist_off, const int64_t *tgt_off, int64_t B, int64_t T, int64_t Nt,
                                  int64_t *bad_index) {
  int64_t dummy;
  if (!bad_index) bad_index = &dummy;
  // the oracle's order: OFFSETS of either array before EMPTY_HISTORY
  stca_status s = check_offsets(hist_off, B, T, false, bad_index);
  if (s != STCA_OK) return s;
  s = check_offsets(tgt_off, B, Nt, false, bad_index);
  if (s != STCA_OK) return s;
  return check_offsets(hist_off, B, T, true, bad_index);
}

void stca_plan_suffix(const int64_t *hist_off, int64_t B, int32_t L_infer, int64_t *start_out) {
  for (int64_t b = 0; b < B; ++b) {
    int64_t s = hist_off[b];
    if (L_infer > 0 && hist_off[b + 1] - L_infer > s) s = hist_off[b + 1] - L_infer;
    start_out[b] = s;
  }
}

int32_t stca_plan_chunks(int64_t L, int32_t chunk_keys, int64_t *chunk_len) {
  const int64_t cap = chunk_keys > 0 ? chunk_keys : STCA_DEFAULT_CHUNK_KEYS;
  if (L <= 0) {
    if (chunk_len) *chunk_len = 0;
    return 0;
  }
  const int64_t n = (L + cap - 1) / cap;
  int64_t cl = (L + n - 1) / n;
  cl = (cl + 127) / 128 * 128;
  if (chunk_len) *chunk_len = cl;
  return (int32_t)((L + cl - 1) / cl);
}

int64_t stca_plan_attention(const int64_t *hist_len, const int64_t *tgt_off, int64_t B, int32_t h, int32_t qtile,
                            int32_t chunk_keys, int64_t *items, int64_t cap) {
  struct It {
    int64_t b, q0, nq, k0, kl, c;
  };
  std::vector<It> v;
  for (int64_t b = 0; b < B; ++b) {
    const int64_t rows = (tgt_off[b + 1] - tgt_off[b]) * h;
    if (rows == 0) continue;
    int64_t cl = 0;
    const int32_t nc = stca_plan_chunks(hist_len[b], chunk_keys, &cl);
    for (int32_t c = 0; c < nc; ++c) {
      const int64_t k0 = (int64_t)c * cl, kl = std::min(cl, hist_len[b] - k0);
      for (int64_t q = 0; q < rows; q += qtile)
        v.push_back({b, tgt_off[b] * h + q, std::min<int64_t>(qtile, rows - q), k0, kl, c});
    }
  }
  // LPT launch order: longest key span first; ties by (request, chunk, query tile)
  std::stable_sort(v.begin(), v.end(), [](const It &a, const It &b) {
    if (a.kl != b.kl) return a.kl > b.kl;
    if (a.b != b.b) return a.b < b.b;
    if (a.c != b.c) return a.c < b.c;
    return a.q0 < b.q0;
  });
  const int64_t n = (int64_t)v.size();
  if (items && n <= cap)
    for (int64_t i = 0; i < n; ++i) {
      int64_t *o = items + 6 * i;
      o[0] = v[i].b; o[1] = v[i].q0; o[2] = v[i].nq; o[3] = v[i].k0; o[4] = v[i].kl; o[5] = v[i].c;
    }
  return n;
}

void stca_plan_split(int64_t L, int32_t chunk_keys, int32_t G, int32_t g, int64_t *own0, int64_t *olen) {
  int64_t cl = 0;
  const int64_t C = stca_plan_chunks(L, chunk_keys, &cl);
  if (G < 1) G = 1;
  const int64_t c0 = ((int64_t)g * C + G - 1) / G, c1 = ((int64_t)(g + 1) * C + G - 1) / G;
  *own0 = std::min(L, c0 * cl);
  *olen = std::min(L, c1 * cl) - *own0;
}

void stca_plan_shards(const int64_t *cost, int64_t B, int32_t n_parts, int32_t *part_out) {
  std::vector<int64_t> idx(B);
  for (int64_t b = 0; b < B; ++b) idx[b] = b;
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
    if (cost[a] != cost[b]) return cost[a] > cost[b];
    return a < b;
  });
  std::vector<int64_t> load(n_parts > 0 ? n_parts : 1, 0);
  for (int64_t b : idx) {
    int32_t best = 0;
    for (int32_t p = 1; p < n_parts; ++p)
      if (load[p] < load[best]) best = p;
    part_out[b] = best;
    load[best] += cost[b];
  }
}

void stca_plan_persistent(const int64_t *cost, int64_t n, int32_t n_ctas, int32_t *cta_list, int32_t *bin_out) {
  if (n_ctas < 1) n_ctas = 1;
  stca_plan_shards(cost, n, n_ctas, bin_out);
  // CSR: cta_list[0 .. n_ctas] offsets, then the items of each CTA in descending cost (stable)
  std::vector<int64_t> idx((size_t)n);
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
    if (bin_out[a] != bin_out[b]) return bin_out[a] < bin_out[b];
    if (cost[a] != cost[b]) return cost[a] > cost[b];
    return a < b;
  });
  int32_t *off = cta_list, *lst = cta_list + n_ctas + 1;
  for (int32_t c = 0; c <= n_ctas; ++c) off[c] = 0;
  for (int64_t i = 0; i < n; ++i) ++off[bin_out[i] + 1];
  for (int32_t c = 0; c < n_ctas; ++c) off[c + 1] += off[c];
  for (int64_t i = 0; i < n; ++i) lst[i] = (int32_t)idx[i];
}

}  // extern "C"

static int32_t *ctal_resize(std::vector<int32_t> &v, int n_ctas, int64_t n) {
  v.assign((size_t)n_ctas + 1 + (size_t)n, 0);
  return v.data();
}

// ===========================================================================
// create / destroy
// ===========================================================================
static bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static void *dalloc(stca_handle *h, size_t bytes) {
  void *p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  h->allocs.push_back(p);
  return p;
}

// Uploads host fp32 `src` into storage dtype; returns device pointer (or null).
static void *upload(stca_handle *h, const float *src, size_t n, bool as_f32 = false) {
  if (!h->bf16 || as_f32) {
    void *p = dalloc(h, n * 4);
    if (p && cudaMemcpy(p, src, n * 4, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    return p;
  }
  std::vector<uint16_t> tmp(n);
  for (size_t i = 0; i < n; ++i) {  // fp32 -> bf16 RNE (storage rounding of the weights)
    uint32_t u;
    memcpy(&u, &src[i], 4);
    tmp[i] = (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
  }
  void *p = dalloc(h, n * 2);
  if (p && cudaMemcpy(p, tmp.data(), n * 2, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  return p;
}

// The weight roles of include/stca.h (names and [rows x cols]), in the order stca_create documents.
struct Need {
  std::string name;
  int64_t rows, cols;
};
static std::vector<Need> weight_roles(int d, int r, int M, bool with_z) {
  const int rd = r * d;
  std::vector<Need> need;
  for (int i = 1; i <= M; ++i) {
    std::string p = "L" + std::to_string(i) + ".";
    need.push_back({p + "hist.Wu", d, rd});
    need.push_back({p + "hist.Wv", d, rd});
    need.push_back({p + "hist.Wo", rd, d});
    need.push_back({p + "hist.ln_g", 1, d});
    need.push_back({p + "hist.ln_b", 1, d});
    need.push_back({p + "qry.Wu", d, rd});
    need.push_back({p + "qry.Wv", d, rd});
    need.push_back({p + "qry.Wo", rd, d});
    if (i == 1) {
      need.push_back({"L1.qry.ln_g", 1, d});
      need.push_back({"L1.qry.ln_b", 1, d});
    }
    for (const char *k : {"WQ", "WK", "WV", "WO"}) need.push_back({p + k, d, d});
    if (i >= 2) need.push_back({p + "WC", (int64_t)i * d, d});
  }
  if (with_z) {
    need.push_back({"z.WZ", (int64_t)(M + 1) * d, d});
    need.push_back({"z.Wu", d, rd});
    need.push_back({"z.Wv", d, rd});
    need.push_back({"z.Wo", rd, d});
  }
  return need;
}

extern "C" stca_status stca_create(const stca_config *cfg, const stca_tensor *w, int32_t n_w, stca_handle **out) {
  if (!cfg || !out || (n_w > 0 && !w)) return STCA_ERR_INVALID_ARG;
  *out = nullptr;
  stca_handle *h = new stca_handle();
  h->cfg = *cfg;
  h->err.clear();
  auto bad = [&](stca_status s) {
    g_create_error = h->err;  // readable through stca_last_error(NULL)
    stca_destroy(h);
    return s;
  };
  const int d = cfg->d, hh = cfg->h, r = cfg->r, M = cfg->M;
  if (d <= 0 || hh <= 0 || r < 1 || M < 1 || M > STCA_MAX_LAYERS || d % hh)
    return bad(fail(h, STCA_ERR_SHAPE, "bad config d=%d h=%d r=%d M=%d (need d%%h==0, r>=1, 1<=M<=%d)", d, hh, r,
                    M, STCA_MAX_LAYERS));
  if (cfg->dtype != STCA_BF16 && cfg->dtype != STCA_FP32) return bad(fail(h, STCA_ERR_INVALID_ARG, "bad dtype"));
  if (cfg->dtype == STCA_BF16 && (d % 16 || d > 512))
    return bad(fail(h, STCA_ERR_UNSUPPORTED, "bf16 path needs d %% 16 == 0 and d <= 512 (d=%d)", d));
  if (cfg->dtype == STCA_FP32 && d > 512) return bad(fail(h, STCA_ERR_UNSUPPORTED, "d <= 512 (d=%d)", d));
  if (cfg->chunk_keys < 0 || cfg->chunk_keys % 128)
    return bad(fail(h, STCA_ERR_INVALID_ARG, "chunk_keys must be a multiple of 128 (got %d)", cfg->chunk_keys));
  if (cfg->split_world < 0 || cfg->split_world > 64 ||
      (cfg->split_world > 1 && (cfg->split_rank < 0 || cfg->split_rank >= cfg->split_world)))
    return bad(fail(h, STCA_ERR_INVALID_ARG, "bad split-history settings (rank %d of %d, exchange %p)",
                    cfg->split_rank, cfg->split_world, (void *)cfg->exchange));
  if (!(cfg->ln_eps > 0.f)) h->cfg.ln_eps = 1e-5f;
  if (h->cfg.split_world == 0) h->cfg.split_world = 1;
  h->bf16 = cfg->dtype == STCA_BF16;
  h->es = h->bf16 ? 2 : 4;
  h->chunk_cap = cfg->chunk_keys > 0 ? cfg->chunk_keys : STCA_DEFAULT_CHUNK_KEYS;
  if ((cfg->dev_alloc == nullptr) != (cfg->dev_free == nullptr))
    return bad(fail(h, STCA_ERR_INVALID_ARG, "dev_alloc and dev_free must both be set or both be NULL"));
  h->al.fa = cfg->dev_alloc;
  h->al.ff = cfg->dev_free;
  h->al.ctx = cfg->alloc_ctx;
  h->al.dev = cfg->device;
  {
    int n = 0;
    DevBuf *const *v = all_bufs(h, &n);
    for (int i = 0; i < n; ++i) v[i]->al = &h->al;
  }
  if (cudaSetDevice(cfg->device) != cudaSuccess) {
    cudaGetLastError();
    return bad(fail(h, STCA_ERR_CUDA, "cudaSetDevice(%d) failed", cfg->device));
  }
  // the bf16 path is tcgen05-only: no CUDA-core substitute for its GEMMs / projection
  if (h->bf16 && !stca::tc_available())
    return bad(fail(h, STCA_ERR_UNSUPPORTED, "the bf16 path needs an sm_100a (B200) device; device %d is not one",
                    cfg->device));

  // ---- collect and validate names / shapes ----
  std::map<std::string, const stca_tensor *> byname;
  for (int i = 0; i < n_w; ++i) {
    if (!w[i].name || !w[i].data) return bad(fail(h, STCA_ERR_INVALID_ARG, "weight %d has a NULL name or data", i));
    if (byname.count(w[i].name)) return bad(fail(h, STCA_ERR_INVALID_ARG, "duplicate weight '%s'", w[i].name));
    byname[w[i].name] = &w[i];
  }
  const int rd = r * d;
  const std::vector<Need> need = weight_roles(d, r, M, cfg->with_z != 0);
  for (const Need &n : need) {
    auto it = byname.find(n.name);
    if (it == byname.end()) return bad(fail(h, STCA_ERR_SHAPE, "missing weight '%s' (%lld x %lld)", n.name.c_str(),
                                            (long long)n.rows, (long long)n.cols));
    if (it->second->rows != n.rows || it->second->cols != n.cols)
      return bad(fail(h, STCA_ERR_SHAPE, "weight '%s' has shape %lld x %lld, expected %lld x %lld", n.name.c_str(),
                      (long long)it->second->rows, (long long)it->second->cols, (long long)n.rows,
                      (long long)n.cols));
  }
  if (byname.size() != need.size()) {
    for (auto &kv : byname) {
      bool ok = false;
      for (const Need &n : need) ok |= n.name == kv.first;
      if (!ok) return bad(fail(h, STCA_ERR_INVALID_ARG, "unknown weight '%s'", kv.first.c_str()));
    }
  }
  auto W = [&](const std::string &n) { return byname[n]->data; };

  // ---- repack ----
  auto ffn = [&](const std::string &p, void **W1, void **Wo, stca::TcWeights *tc) -> bool {
    const float *u = W(p + ".Wu"), *v = W(p + ".Wv"), *o = W(p + ".Wo");
    std::vector<float> il((size_t)d * 2 * rd);
    for (int e = 0; e < d; ++e)
      for (int j = 0; j < rd; ++j) {
        il[(size_t)e * 2 * rd + 2 * j] = u[(size_t)e * rd + j];
        il[(size_t)e * 2 * rd + 2 * j + 1] = v[(size_t)e * rd + j];
      }
    *W1 = upload(h, il.data(), il.size());
    *Wo = upload(h, o, (size_t)rd * d);
    if (!*W1 || !*Wo) return false;
    if (tc && h->bf16 && !stca::tc_prepare_ffn(u, v, o, d, rd, tc, [&](size_t n) { return dalloc(h, n); }))
      return false;
    return true;
  };
  const float qk_scale = (float)(1.4426950408889634 / sqrt((double)(d / hh)));  // log2(e)/sqrt(d_h)
  float *wq = (float *)dalloc(h, (size_t)d * d * 4), *wk = (float *)dalloc(h, (size_t)d * d * 4);
  float *wv = (float *)dalloc(h, (size_t)d * d * 4), *wo = (float *)dalloc(h, (size_t)d * d * 4);
  float *wqk = (float *)dalloc(h, (size_t)hh * d * d * 4), *wvo = (float *)dalloc(h, (size_t)hh * d * d * 4);
  if (!wq || !wk || !wv || !wo || !wqk || !wvo) return bad(fail(h, STCA_ERR_OOM, "weight staging allocation failed"));
  for (int i = 1; i <= M; ++i) {
    LayerW &Ly = h->L[i - 1];
    std::string p = "L" + std::to_string(i) + ".";
    if (!ffn(p + "hist", &Ly.W1h, &Ly.Woh, &Ly.tc)) return bad(fail(h, STCA_ERR_OOM, "upload failed (%s)", p.c_str()));
    {  // [Wu | Wv] column blocks, bf16 [d x 2rd]: the history backward's recompute and dX GEMMs
      const float *u = W(p + "hist.Wu"), *v = W(p + "hist.Wv");
      std::vector<float> cat((size_t)d * 2 * rd);
      for (int e = 0; e < d; ++e) {
        memcpy(&cat[(size_t)e * 2 * rd], u + (size_t)e * rd, sizeof(float) * rd);
        memcpy(&cat[(size_t)e * 2 * rd + rd], v + (size_t)e * rd, sizeof(float) * rd);
      }
      if (!(Ly.W1cat = upload(h, cat.data(), cat.size())))
        return bad(fail(h, STCA_ERR_OOM, "upload failed (%shist.Wu/Wv)", p.c_str()));
    }
    if (W(p + "qry.Wu") == W(p + "hist.Wu") && W(p + "qry.Wv") == W(p + "hist.Wv") && W(p + "qry.Wo") == W(p + "hist.Wo")) {
      Ly.W1q = Ly.W1h;
      Ly.Woq = Ly.Woh;
      Ly.tc.W1q = Ly.tc.W1h;
      Ly.tc.Woq = Ly.tc.Woh;
    } else {
      stca::TcWeights tq;
      if (!ffn(p + "qry", &Ly.W1q, &Ly.Woq, &tq)) return bad(fail(h, STCA_ERR_OOM, "upload failed (%sqry)", p.c_str()));
      Ly.tc.W1q = tq.W1h;
      Ly.tc.Woq = tq.Woh;
    }
    Ly.gh = (float *)upload(h, W(p + "hist.ln_g"), d, true);
    Ly.bh = (float *)upload(h, W(p + "hist.ln_b"), d, true);
    if (i == 1) {
      Ly.gq = (float *)upload(h, W("L1.qry.ln_g"), d, true);
      Ly.bq = (float *)upload(h, W("L1.qry.ln_b"), d, true);
    }
    // W_QK, W_VO on the device (fp32), then storage dtype
    if (cudaMemcpy(wq, W(p + "WQ"), (size_t)d * d * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(wk, W(p + "WK"), (size_t)d * d * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(wv, W(p + "WV"), (size_t)d * d * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(wo, W(p + "WO"), (size_t)d * d * 4, cudaMemcpyHostToDevice) != cudaSuccess)
      return bad(fail(h, STCA_ERR_CUDA, "weight upload failed"));
    if (stca::prep_qk_vo(wq, wk, wv, wo, d, hh, qk_scale, wqk, wvo, 0) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
      return bad(fail(h, STCA_ERR_CUDA, "prep_qk_vo failed: %s", cudaGetErrorString(cudaGetLastError())));
    const size_t nqk = (size_t)hh * d * d;
    if (h->bf16) {
      Ly.WQK = dalloc(h, nqk * 2);
      Ly.WVO = dalloc(h, nqk * 2);
      if (!Ly.WQK || !Ly.WVO) return bad(fail(h, STCA_ERR_OOM, "alloc failed"));
      stca::f32_to_bf16(wqk, (bf16 *)Ly.WQK, nqk, 0);
      stca::f32_to_bf16(wvo, (bf16 *)Ly.WVO, nqk, 0);
    } else {
      Ly.WQK = dalloc(h, nqk * 4);
      Ly.WVO = dalloc(h, nqk * 4);
      if (!Ly.WQK || !Ly.WVO) return bad(fail(h, STCA_ERR_OOM, "alloc failed"));
      cudaMemcpy(Ly.WQK, wqk, nqk * 4, cudaMemcpyDeviceToDevice);
      cudaMemcpy(Ly.WVO, wvo, nqk * 4, cudaMemcpyDeviceToDevice);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return bad(fail(h, STCA_ERR_CUDA, "weight prep failed"));
    if (i >= 2) {  // permute rows: [o1..o(i-1) | x_t] -> Ocat layout [x_t | o1 | .. | o(i-1)]
      const float *wc = W(p + "WC");
      std::vector<float> pc((size_t)i * d * d);
      memcpy(pc.data(), wc + (size_t)(i - 1) * d * d, sizeof(float) * d * d);
      memcpy(pc.data() + (size_t)d * d, wc, sizeof(float) * (size_t)(i - 1) * d * d);
      Ly.WC = upload(h, pc.data(), pc.size());
      if (!Ly.WC) return bad(fail(h, STCA_ERR_OOM, "alloc failed"));
    }
    if (h->bf16 && !stca::tc_prepare_layer(Ly.WQK, Ly.WVO, Ly.WC, i, d, hh, &Ly.tc, [&](size_t n) { return dalloc(h, n); }))
      return bad(fail(h, STCA_ERR_OOM, "tc repack failed"));
  }
  if (h->bf16) {
    std::vector<const float *> wu(M), wv(M), wo_(M), gg(M), bb(M);
    for (int i = 0; i < M; ++i) {
      std::string p = "L" + std::to_string(i + 1) + ".hist.";
      wu[i] = W(p + "Wu");
      wv[i] = W(p + "Wv");
      wo_[i] = W(p + "Wo");
      gg[i] = W(p + "ln_g");
      bb[i] = W(p + "ln_b");
    }
    if (!stca::tc_prepare_proj(wu.data(), wv.data(), wo_.data(), gg.data(), bb.data(), M, d, rd, &h->tcp,
                               [&](size_t n) { return dalloc(h, n); }))
      return bad(fail(h, STCA_ERR_OOM, "projection weight repack failed"));
  }
  if (cfg->with_z) {
    if (!ffn("z", &h->W1z, &h->Woz, &h->tcz)) return bad(fail(h, STCA_ERR_OOM, "upload failed (z)"));
    const float *wz = W("z.WZ");
    std::vector<float> pz((size_t)(M + 1) * d * d);
    memcpy(pz.data(), wz + (size_t)M * d * d, sizeof(float) * d * d);
    memcpy(pz.data() + (size_t)d * d, wz, sizeof(float) * (size_t)M * d * d);
    h->WZ = upload(h, pz.data(), pz.size());
    if (!h->WZ) return bad(fail(h, STCA_ERR_OOM, "alloc failed"));
    if (h->bf16 && !stca::tc_prepare_layer(nullptr, nullptr, h->WZ, M + 1, d, hh, &h->tcz, [&](size_t n) { return dalloc(h, n); }))
      return bad(fail(h, STCA_ERR_OOM, "tc repack failed"));
  }
  if (h->bf16 && d == 128) {  // the whole-stack backward (stca_backward) works on fp32 target-side weights
    for (const Need &n : need) {
      if (n.name.find(".hist.") != std::string::npos) continue;
      float *p = (float *)upload(h, W(n.name), (size_t)(n.rows * n.cols), true);
      if (!p) return bad(fail(h, STCA_ERR_OOM, "upload failed (%s)", n.name.c_str()));
      h->w32[n.name] = p;
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return bad(fail(h, STCA_ERR_CUDA, "create: device error"));
  *out = h;
  return STCA_OK;
}

extern "C" void stca_destroy(stca_handle *h) {
  if (!h) return;
  cudaSetDevice(h->cfg.device);
  cudaDeviceSynchronize();
  for (void *p : h->allocs) cudaFree(p);
  if (h->peer_buf) cudaFree(h->peer_buf);
  if (h->peer_tab) cudaFree(h->peer_tab);
  int nb = 0;
  DevBuf *const *bufs = all_bufs(h, &nb);
  for (int i = 0; i < nb; ++i) bufs[i]->release();
  cudaDeviceSynchronize();  // stream-ordered frees on the legacy stream
  h->stage.release();
  stca::hist_bwd_release(h->blas);
  for (ProfRegion &r : h->prof_open) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : h->prof_pool) cudaEventDestroy(e);
  if (h->copy_st) {
    cudaStreamDestroy(h->copy_st);
    for (cudaEvent_t e : h->ev_xin_free) cudaEventDestroy(e);
    cudaEventDestroy(h->ev_xtin_free);
    cudaEventDestroy(h->ev_xt_in);
    for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
  }
  cudaGetLastError();
  delete h;
}

extern "C" const char *stca_last_error(const stca_handle *h) { return h ? h->err.c_str() : g_create_error.c_str(); }

// A pinned (host-mapped) staging slot of at least `bytes` bytes for uploads enqueued on `st`; the
// caller records *ev on `st` after the upload.  Waits only if the slot's previous upload is unfinished.
static stca_status staging_acquire(stca_handle *h, size_t bytes, void **out, cudaEvent_t *ev) {
  StagingRing &r = h->stage;
  const int k = r.next;
  r.next = (k + 1) % STAGING_SLOTS;
  if (!r.ev[k]) CU(cudaEventCreateWithFlags(&r.ev[k], cudaEventDisableTiming));
  CU(cudaEventSynchronize(r.ev[k]));  // the slot's last copy has read it (normally long done)
  CU(r.buf[k].ensure(bytes));
  *out = r.buf[k].p;
  *ev = r.ev[k];
  return STCA_OK;
}

// ===========================================================================
// project_history
// ===========================================================================
// a1: X~(i) = LN(SwiGLUFFN(i)(X)) for all layers, Eq.(2), for cache rows [r0, r0 + rows) (X points at
// row r0 of the compacted input)
// The handle's copy stream for host inputs (created on first use; its "buffer free" events are
// recorded on `st` right away, so the first uploads wait for every earlier reader on `st`).
static stca_status ensure_copy_stream(stca_handle *h, cudaStream_t st) {
  if (h->copy_st) return STCA_OK;
  CU(cudaStreamCreateWithFlags(&h->copy_st, cudaStreamNonBlocking));
  for (cudaEvent_t &e : h->ev_xin_free) {
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CU(cudaEventRecord(e, st));
  }
  CU(cudaEventCreateWithFlags(&h->ev_xtin_free, cudaEventDisableTiming));
  CU(cudaEventRecord(h->ev_xtin_free, st));
  CU(cudaEventCreateWithFlags(&h->ev_xt_in, cudaEventDisableTiming));
  for (cudaEvent_t &e : h->ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return STCA_OK;
}

// Host plan -> device buffer `dst` through a staging slot and a fetch kernel on `st` (SM loads of
// mapped pinned memory): never queued behind a large host-input copy in the H2D copy engine.
static stca_status upload_plan(stca_handle *h, const void *src, size_t bytes, DevBuf &dst, cudaStream_t st) {
  const size_t b16 = (bytes + 15) / 16 * 16;
  CU(dst.ensure(b16 + 64, st));
  if (!bytes) return STCA_OK;
  void *slot = nullptr;
  cudaEvent_t slot_ev = nullptr;
  stca_status s = staging_acquire(h, b16, &slot, &slot_ev);
  if (s != STCA_OK) return s;
  memcpy(slot, src, bytes);
  CU(stca::fetch_mapped(slot, dst.p, b16, st));
  CU(cudaEventRecord(slot_ev, st));
  return STCA_OK;
}

static stca_status project_rows(stca_handle *h, const void *X, int64_t r0, int64_t rows, cudaStream_t st) {
  const int d = h->cfg.d, M = h->cfg.M, rd = h->cfg.r * d, es = h->es;
  const size_t row_bytes = (size_t)d * es;
  const int64_t T2 = h->T2;
  if (h->bf16) {  // tcgen05 (stca_create refused bf16 without an sm_100a device)
    stca::TcProj pj;
    pj.X = X;
    pj.rows = rows;
    pj.d = d;
    pj.rd = rd;
    pj.M = M;
    pj.eps = h->cfg.ln_eps;
    pj.out = (uint8_t *)h->xt_cache.p + (size_t)r0 * row_bytes;
    pj.out_layer_stride = T2 * d;
    pj.W1cat = h->tcp.W1cat;
    pj.Wocat = h->tcp.Wocat;
    pj.gcat = h->tcp.gcat;
    pj.bcat = h->tcp.bcat;
    for (int i = 0; i < M; ++i) {
      pj.W1[i] = h->L[i].tc.W1h;
      pj.Wo[i] = h->L[i].tc.Woh;
      pj.g[i] = h->L[i].gh;
      pj.b[i] = h->L[i].bh;
    }
    if (d != 128) {  // two-GEMM path: the handle's H scratch, pieces of at most 2^18 rows
      pj.H_rows = std::min<int64_t>(rows, 1 << 18);
      CU(h->proj_h.ensure((size_t)pj.H_rows * rd * 2, st));
      pj.H = h->proj_h.p;
    }
    cudaEvent_t pa = prof_begin(h, st);
    for (int rep = 0; rep < h->reps_proj; ++rep) CU(stca::tc_project(pj, st));  // idempotent
    prof_end(h, STCA_PH_PROJECT, pa, st);
    return STCA_OK;
  }
  const int64_t R = std::min<int64_t>(std::max<int64_t>(rows, 1), 1 << 16);
  CU(h->proj_h.ensure((size_t)R * rd * es, st));
  CU(h->proj_y.ensure((size_t)R * d * 4, st));
  for (int i = 0; i < M; ++i) {
    for (int64_t q0 = 0; q0 < rows; q0 += R) {
      const int n = (int)std::min<int64_t>(R, rows - q0);
      const uint8_t *xa = (const uint8_t *)X + (size_t)q0 * row_bytes;
      CU(stca::cc_gemm(h->bf16, xa, d, h->L[i].W1h, 2 * rd, h->proj_h.p, rd, nullptr, 0, n, 2 * rd, d, 1.f,
                       stca::EPI_SWIGLU, st));
      CU(stca::cc_gemm(h->bf16, h->proj_h.p, rd, h->L[i].Woh, d, nullptr, 0, h->proj_y.as<float>(), d, n, d, rd,
                       1.f, stca::EPI_STORE, st));
      uint8_t *dst = (uint8_t *)h->xt_cache.p + ((size_t)i * T2 + r0 + q0) * row_bytes;
      CU(stca::cc_layernorm(h->bf16, h->proj_y.as<float>(), d, h->L[i].gh, h->L[i].bh, h->cfg.ln_eps, dst, d, n, d,
                            st));
    }
  }
  return STCA_OK;
}

// validation of a projection call (nothing is enqueued on failure): offsets, empty histories, the
// split-K fold's chunk limit
static stca_status validate_history(stca_handle *h, const void *X, int64_t T, const int64_t *hist_off, int64_t B) {
  if (h->sticky) return fail(h, STCA_ERR_CUDA, "handle is in a sticky CUDA error state: %s", h->err.c_str());
  if (B < 0 || T < 0 || !hist_off || (T > 0 && !X)) return fail(h, STCA_ERR_INVALID_ARG, "NULL or negative argument");
  int64_t badi = -1;
  stca_status s = check_offsets(hist_off, B, T, false, &badi);
  if (s != STCA_OK) return fail(h, s, "hist_off invalid at request %lld (off[0]=%lld, off[B]=%lld, T=%lld)",
                                (long long)badi, (long long)hist_off[0], (long long)hist_off[B], (long long)T);
  s = check_offsets(hist_off, B, T, true, &badi);
  if (s != STCA_OK) return fail(h, s, "empty history for request %lld", (long long)badi);
  for (int64_t b = 0; b < B; ++b) {  // the split-K merge folds at most 8 chunks per history
    int64_t Lb = hist_off[b + 1] - hist_off[b];
    if (h->cfg.L_infer > 0 && Lb > h->cfg.L_infer) Lb = h->cfg.L_infer;
    if (stca_plan_chunks(Lb, (int32_t)h->chunk_cap, nullptr) > 8)
      return fail(h, STCA_ERR_UNSUPPORTED, "history %lld has %lld keys > 8 x chunk_keys (%lld); raise chunk_keys",
                  (long long)b, (long long)Lb, (long long)h->chunk_cap);
  }
  return STCA_OK;
}

extern "C" stca_status stca_project_history(stca_handle *h, const void *X, int64_t T, const int64_t *hist_off,
                                            int64_t B, void *stream) {
  if (!h) return STCA_ERR_INVALID_ARG;
  stca_status s = validate_history(h, X, T, hist_off, B);
  if (s != STCA_OK) return s;
  h->sess_on = false;  // a plain projection replaces any session cache (its entries are forgotten)
  h->sess.clear();
  h->sess_pos.clear();
  CU(cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  const int d = h->cfg.d, M = h->cfg.M, es = h->es;
  const size_t row_bytes = (size_t)d * es;
  h->B = -1;  // no valid projection until this call has enqueued all of its work (a failure below leaves none)

  // a0: suffix truncation + compacted offsets (exact integer work)
  h->start.assign(B, 0);
  stca_plan_suffix(hist_off, B, h->cfg.L_infer, h->start.data());
  h->len.assign(B, 0);
  h->own0.assign(B, 0);
  h->olen.assign(B, 0);
  h->coff.assign(B + 1, 0);
  bool gather = false;
  const int G = h->cfg.split_world, g = h->cfg.split_rank;
  for (int64_t b = 0; b < B; ++b) {
    h->len[b] = hist_off[b + 1] - h->start[b];
    h->olen[b] = h->len[b];
    if (G > 1)  // split-history: this rank owns chunks [ceil(g C / G), ceil((g+1) C / G)) of the history
      stca_plan_split(h->len[b], (int32_t)h->chunk_cap, G, g, &h->own0[b], &h->olen[b]);
    h->coff[b + 1] = h->coff[b] + h->olen[b];
    gather |= h->start[b] + h->own0[b] != hist_off[b] || h->olen[b] != hist_off[b + 1] - hist_off[b];
  }
  const int64_t T2 = h->coff[B];  // rows of the X~ cache (the suffix rows this rank owns)
  CU(h->xt_cache.ensure((size_t)M * T2 * row_bytes + 256, st));
  h->T2 = T2;
  const void *Xd = X;
  const bool host_x = T > 0 && !is_device_ptr(X);
  if (host_x && !gather && T2 > 0) {
    // host input, no gather: stream X up in pieces on a copy stream and project each piece as soon as
    // it has landed, so the H2D copy (the e2e bottleneck) overlaps the projection of earlier pieces
    stca_status cs = ensure_copy_stream(h, st);
    if (cs != STCA_OK) return cs;
    // two staging buffers in turn: the upload of call n + 1 waits only for the projection of call n - 1
    // (its buffer's last reader), so the PCIe copies of consecutive calls run back to back
    const int xk = h->xin_k;
    h->xin_k ^= 1;
    DevBuf &xin = h->xin[xk];
    void *const xin_old = xin.p;
    CU(xin.ensure((size_t)T * row_bytes, st));
    // a regrown buffer was allocated in `stream` order: the copy stream may write it only after that point
    if (xin.p != xin_old) CU(cudaEventRecord(h->ev_xin_free[xk], st));
    CU(cudaStreamWaitEvent(h->copy_st, h->ev_xin_free[xk], 0));
    const int npieces = (int)std::min<int64_t>(STCA_H2D_PIECES, (T2 + (1 << 16) - 1) >> 16);
    const int64_t step = ((T2 + npieces - 1) / npieces + 255) / 256 * 256;  // whole 128-row tile pairs
    int k = 0;
    for (int64_t r0 = 0; r0 < T2; r0 += step, ++k) {
      const int64_t rows = std::min<int64_t>(step, T2 - r0);
      uint8_t *dst = (uint8_t *)xin.p + (size_t)r0 * row_bytes;
      CU(cudaMemcpyAsync(dst, (const uint8_t *)X + (size_t)r0 * row_bytes, (size_t)rows * row_bytes,
                         cudaMemcpyHostToDevice, h->copy_st));
      CU(cudaEventRecord(h->ev[k], h->copy_st));
      CU(cudaStreamWaitEvent(st, h->ev[k], 0));
      stca_status s = project_rows(h, dst, r0, rows, st);
      if (s != STCA_OK) return s;
    }
    CU(cudaEventRecord(h->ev_xin_free[xk], st));
    h->B = B;
    return STCA_OK;
  }
  if (host_x) {  // host input with a gather: stage all of X on the stream first
    // on `stream` itself (ordered after every earlier reader); the copy stream's next upload into this
    // buffer is ordered after this call's projection by ev_xin_free below
    CU(h->xin[0].ensure((size_t)T * row_bytes, st));
    CU(cudaMemcpyAsync(h->xin[0].p, X, (size_t)T * row_bytes, cudaMemcpyHostToDevice, st));
    Xd = h->xin[0].p;
  }
  if (gather && T2 > 0) {  // gather the (owned) suffix rows into a compacted buffer
    std::vector<int64_t> seg;
    int64_t maxlen = 0;
    for (int64_t b = 0; b < B; ++b) {
      seg.push_back(h->start[b] + h->own0[b]);
      seg.push_back(h->coff[b]);
      seg.push_back(h->olen[b]);
      maxlen = std::max(maxlen, h->olen[b]);
    }
    stca_status ss = upload_plan(h, seg.data(), seg.size() * 8, h->seg, st);
    if (ss != STCA_OK) return ss;
    CU(h->xgather.ensure((size_t)T2 * row_bytes, st));
    CU(stca::gather_rows(Xd, h->xgather.p, h->seg.as<int64_t>(), B, maxlen, (int)row_bytes, st));
    Xd = h->xgather.p;
  }
  if (T2 > 0) {
    stca_status s = project_rows(h, Xd, 0, T2, st);
    if (s != STCA_OK) return s;
  }
  if (host_x && h->ev_xin_free[0]) CU(cudaEventRecord(h->ev_xin_free[0], st));
  h->B = B;
  return STCA_OK;
}

// ===========================================================================
// session sharing (NEXT-4): RLB extended across requests of the same user
// ===========================================================================
extern "C" stca_status stca_session_open(stca_handle *h, int64_t capacity_rows, void *stream) {
  if (!h) return STCA_ERR_INVALID_ARG;
  if (h->sticky) return fail(h, STCA_ERR_CUDA, "handle is in a sticky CUDA error state: %s", h->err.c_str());
  if (capacity_rows < 1) return fail(h, STCA_ERR_INVALID_ARG, "capacity_rows must be >= 1");
  if (h->cfg.split_world > 1) return fail(h, STCA_ERR_UNSUPPORTED, "no session cache in split-history mode");
  CU(cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  h->B = -1;
  CU(h->xt_cache.ensure((size_t)h->cfg.M * capacity_rows * h->cfg.d * h->es + 256, st));
  h->sess_on = true;
  h->sess_cap = capacity_rows;
  h->sess_head = 0;
  h->sess.clear();
  h->sess_pos.clear();
  h->T2 = capacity_rows;  // rows per layer of the cache
  return STCA_OK;
}

extern "C" stca_status stca_project_history_session(stca_handle *h, const int64_t *user_id, const int64_t *gen,
                                                    const void *X, int64_t T, const int64_t *hist_off, int64_t B,
                                                    int64_t *n_projected, void *stream) {
  if (!h) return STCA_ERR_INVALID_ARG;
  if (!h->sess_on) return fail(h, STCA_ERR_STATE, "stca_project_history_session before stca_session_open");
  if (B > 0 && (!user_id || !gen)) return fail(h, STCA_ERR_INVALID_ARG, "user_id / gen is NULL");
  stca_status s = validate_history(h, X, T, hist_off, B);
  if (s != STCA_OK) return s;
  // a0: the temporal suffix of every request
  std::vector<int64_t> start(B), len(B);
  stca_plan_suffix(hist_off, B, h->cfg.L_infer, start.data());
  int64_t total = 0;
  for (int64_t b = 0; b < B; ++b) {
    len[b] = hist_off[b + 1] - start[b];
    total += len[b];
  }
  // Hits: (user, generation, kept length) in the cache; a user twice in one batch with the same key
  // shares one entry.  The misses get ONE contiguous range of the FIFO ring (one projection launch);
  // entries it overlaps are evicted.  If that would evict a hit of this batch, the cache is reset and
  // the whole batch projected from row 0.
  std::vector<int64_t> miss;  // first request of every missing user, in request order
  int64_t a = 0, R = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (attempt == 1) {
      h->sess.clear();
      h->sess_pos.clear();
      h->sess_head = 0;
    }
    miss.clear();
    R = 0;
    std::map<int64_t, int64_t> hit_users, miss_users;
    for (int64_t b = 0; b < B; ++b) {
      const int64_t u = user_id[b];
      auto it = h->sess.find(u);
      const bool cached = it != h->sess.end() && it->second.gen == gen[b] && it->second.len == len[b];
      auto mu = miss_users.find(u);
      if (mu != miss_users.end()) {  // already missing in this batch: must be the same (gen, length)
        if (gen[mu->second] != gen[b] || len[mu->second] != len[b])
          return fail(h, STCA_ERR_INVALID_ARG, "user %lld appears twice in the batch with different histories",
                      (long long)u);
      } else if (cached) {
        hit_users[u] = b;
      } else {
        miss_users[u] = b;
        miss.push_back(b);
        R += len[b];
      }
    }
    for (auto &hu : hit_users)
      if (miss_users.count(hu.first)) return fail(h, STCA_ERR_INVALID_ARG, "user %lld appears twice in the batch "
                                                  "with different histories", (long long)hu.first);
    if (R > h->sess_cap)
      return fail(h, STCA_ERR_OOM, "the batch needs %lld new cache rows, capacity %lld", (long long)R,
                  (long long)h->sess_cap);
    a = h->sess_head + R <= h->sess_cap ? h->sess_head : 0;
    std::vector<int64_t> evict;
    bool hit_evicted = false;
    for (auto &p : h->sess_pos) {
      const auto &e = h->sess[p.second];
      if (R > 0 && e.off < a + R && e.off + e.len > a) {
        evict.push_back(p.second);
        hit_evicted |= hit_users.count(p.second) > 0;
      }
    }
    if (hit_evicted && attempt == 0) continue;  // reset and project the whole batch
    for (int64_t u : evict) {
      h->sess_pos.erase(h->sess[u].off);
      h->sess.erase(u);
    }
    int64_t off = a;
    for (int64_t b : miss) {  // (re)place every missing user's entry
      auto it = h->sess.find(user_id[b]);
      if (it != h->sess.end()) {
        h->sess_pos.erase(it->second.off);
        h->sess.erase(it);
      }
      h->sess[user_id[b]] = {gen[b], len[b], off};
      h->sess_pos[off] = user_id[b];
      off += len[b];
    }
    h->sess_head = a + R;
    break;
  }
  (void)total;
  CU(cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t row_bytes = (size_t)h->cfg.d * h->es;
  h->B = -1;
  h->start = start;
  h->len = len;
  h->olen = len;
  h->own0.assign(B, 0);
  h->coff.assign(B + 1, 0);
  for (int64_t b = 0; b < B; ++b) h->coff[b] = h->sess[user_id[b]].off;  // key rows of request b in the cache
  h->coff[B] = h->sess_cap;
  h->T2 = h->sess_cap;
  if (R > 0) {  // gather the missing users' suffix rows, project them into cache rows [a, a + R)
    const void *Xd = X;
    if (!is_device_ptr(X)) {
      CU(h->xin[0].ensure((size_t)T * row_bytes, st));
      CU(cudaMemcpyAsync(h->xin[0].p, X, (size_t)T * row_bytes, cudaMemcpyHostToDevice, st));
      Xd = h->xin[0].p;
    }
    std::vector<int64_t> seg;
    int64_t maxlen = 0, dst = 0;
    for (int64_t b : miss) {
      seg.push_back(start[b]);
      seg.push_back(dst);
      seg.push_back(len[b]);
      dst += len[b];
      maxlen = std::max(maxlen, len[b]);
    }
    s = upload_plan(h, seg.data(), seg.size() * 8, h->seg, st);
    if (s != STCA_OK) return s;
    CU(h->xgather.ensure((size_t)R * row_bytes, st));
    CU(stca::gather_rows(Xd, h->xgather.p, h->seg.as<int64_t>(), (int64_t)miss.size(), maxlen, (int)row_bytes, st));
    s = project_rows(h, h->xgather.p, a, R, st);
    if (s != STCA_OK) return s;
    if (h->ev_xin_free[0]) CU(cudaEventRecord(h->ev_xin_free[0], st));
  }
  if (n_projected) *n_projected = (int64_t)miss.size();
  h->B = B;
  return STCA_OK;
}

// ===========================================================================
// forward
// ===========================================================================
static stca_status ffn_rows(stca_handle *h, const void *in, int64_t ldi, int64_t rows, void *W1, void *Wo,
                            const stca::TcWeights *tcw, int which, const float *g, const float *b, void *out_s,
                            int64_t ldo, float *out_f, int64_t ldof, cudaStream_t st) {
  // SwiGLUFFN (+ LN when g != null) on `rows` rows: the query-side instances of Eq.(1), (3), (7), (9)
  const int d = h->cfg.d, rd = h->cfg.r * d, es = h->es;
  if (rows <= 0) return STCA_OK;
  if (h->bf16) {
    CU(h->hbuf.ensure((size_t)rows * rd * 2, st));  // H scratch owned by this handle
    cudaEvent_t pa = h->prof_target ? prof_begin(h, st) : nullptr;
    CU(stca::tc_ffn(in, ldi, rows, which == 0 ? tcw->W1h : tcw->W1q, which == 0 ? tcw->Woh : tcw->Woq, d, rd, g, b,
                    h->cfg.ln_eps, out_s, ldo, out_f, ldof, h->hbuf.p, st));
    prof_end(h, STCA_PH_TARGET, pa, st);
    return STCA_OK;
  }
  CU(h->hbuf.ensure((size_t)rows * rd * es, st));
  CU(h->ybuf32.ensure((size_t)rows * d * 4, st));
  CU(stca::cc_gemm(h->bf16, in, ldi, W1, 2 * rd, h->hbuf.p, rd, nullptr, 0, (int)rows, 2 * rd, d, 1.f,
                   stca::EPI_SWIGLU, st));
  if (g) {
    CU(stca::cc_gemm(h->bf16, h->hbuf.p, rd, Wo, d, nullptr, 0, h->ybuf32.as<float>(), d, (int)rows, d, rd, 1.f,
                     stca::EPI_STORE, st));
    CU(stca::cc_layernorm(h->bf16, h->ybuf32.as<float>(), d, g, b, h->cfg.ln_eps, out_s, ldo, rows, d, st));
  } else {
    CU(stca::cc_gemm(h->bf16, h->hbuf.p, rd, Wo, d, out_s, ldo, out_f, ldof, (int)rows, d, rd, 1.f, stca::EPI_STORE,
                     st));
  }
  return STCA_OK;
}

static stca_status gemm(stca_handle *h, const void *A, int64_t lda, const void *Bw, const void *Btc, int64_t ldb,
                        void *Cs, int64_t ldcs, float *Cf, int64_t ldcf, int64_t M, int N, int K, cudaStream_t st) {
  if (M <= 0) return STCA_OK;
  if (h->bf16) {
    cudaEvent_t pa = h->prof_target ? prof_begin(h, st) : nullptr;
    CU(stca::tc_gemm(A, lda, Btc, M, N, K, Cs, ldcs, Cf, ldcf, st));
    prof_end(h, STCA_PH_TARGET, pa, st);
    return STCA_OK;
  }
  CU(stca::cc_gemm(h->bf16, A, lda, Bw, ldb, Cs, ldcs, Cf, ldcf, (int)M, N, K, 1.f, stca::EPI_STORE, st));
  return STCA_OK;
}

// ===========================================================================
// read back the projected cache (inspection / tests of the history path alone)
// ===========================================================================
extern "C" stca_status stca_read_cache(stca_handle *h, int32_t layer, int64_t row0, int64_t nrows, float *out,
                                       void *stream) {
  if (!h) return STCA_ERR_INVALID_ARG;
  if (h->sticky) return fail(h, STCA_ERR_CUDA, "handle is in a failed state: %s", h->err.c_str());
  if (h->B < 0) return fail(h, STCA_ERR_STATE, "read_cache before project_history");
  if (layer < 1 || layer > h->cfg.M) return fail(h, STCA_ERR_INVALID_ARG, "layer %d outside 1..%d", layer, h->cfg.M);
  if (row0 < 0 || nrows < 0 || row0 + nrows > h->T2)
    return fail(h, STCA_ERR_INVALID_ARG, "rows [%lld, %lld) outside the cache's %lld rows", (long long)row0,
                (long long)(row0 + nrows), (long long)h->T2);
  if (nrows == 0) return STCA_OK;
  if (!out) return fail(h, STCA_ERR_INVALID_ARG, "out is NULL");
  CU(cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  const int d = h->cfg.d;
  const size_t n = (size_t)nrows * d;
  const uint8_t *src = (const uint8_t *)h->xt_cache.p + ((size_t)(layer - 1) * h->T2 + row0) * d * h->es;
  const bool host = !is_device_ptr(out);
  float *dst = out;
  if (host) {
    CU(h->Zout.ensure(n * 4, st));
    dst = h->Zout.as<float>();
  }
  if (h->bf16)
    CU(stca::bf16_to_f32((const stca::bf16 *)src, dst, (int64_t)n, st));
  else
    CU(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyDeviceToDevice, st));
  if (host) {
    CU(cudaMemcpyAsync(out, dst, n * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));  // the scratch buffer is reused by forward
  }
  return STCA_OK;
}

static stca_status forward_body(stca_handle *h, const void *xt, int64_t Nt, const int64_t *tgt_off, int64_t B,
                                float *out_Z, float *out_z, cudaStream_t st);

extern "C" stca_status stca_forward(stca_handle *h, const void *xt, int64_t Nt, const int64_t *tgt_off, int64_t B,
                                    float *out_Z, float *out_z, void *stream) {
  if (!h) return STCA_ERR_INVALID_ARG;
  if (h->sticky) return fail(h, STCA_ERR_CUDA, "handle is in a sticky CUDA error state: %s", h->err.c_str());
  if (h->B < 0) return fail(h, STCA_ERR_STATE, "stca_forward before stca_project_history");
  if (B != h->B) return fail(h, STCA_ERR_STATE, "B=%lld differs from the projected B=%lld", (long long)B, (long long)h->B);
  if (Nt < 0 || !tgt_off || (Nt > 0 && (!xt || !out_Z)))
    return fail(h, STCA_ERR_INVALID_ARG, "NULL or negative argument");
  if (out_z && !h->cfg.with_z) return fail(h, STCA_ERR_INVALID_ARG, "out_z given but the handle has with_z = 0");
  int64_t badi = -1;
  stca_status s = check_offsets(tgt_off, B, Nt, false, &badi);
  if (s != STCA_OK) return fail(h, s, "tgt_off invalid at request %lld (off[B]=%lld, Nt=%lld)", (long long)badi,
                                (long long)tgt_off[B], (long long)Nt);
  if (Nt == 0) return STCA_OK;
  CU(cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t p_fwd = prof_begin(h, st);
  s = forward_body(h, xt, Nt, tgt_off, B, out_Z, out_z, st);
  if (s == STCA_OK) prof_end(h, STCA_PH_FORWARD, p_fwd, st);
  return s;
}

// Split-history epoch exchange as STREAM memory operations (cuStreamWriteValue64 into every peer's flag
// word -- preceded by a system-wide fence of this stream's earlier writes -- then cuStreamWaitValue64 on
// this rank's own flag words): the stream front end waits, no SM is held spinning.  False when the driver
// does not offer them (the caller then launches k_peer_exchange).
typedef CUresult (*MemOp64Fn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
static bool peer_exchange_memops(stca_handle *h, uint64_t epoch, cudaStream_t st) {
  static MemOp64Fn wr = nullptr, wt = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr, *q = nullptr;
    cudaDriverEntryPointQueryResult r1, r2;
    if (getenv("STCA_PEER_KERNEL")) return;  // A/B: the one-thread spinning kernel instead
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &r1) == cudaSuccess &&
        r1 == cudaDriverEntryPointSuccess &&
        cudaGetDriverEntryPoint("cuStreamWaitValue64", &q, cudaEnableDefault, &r2) == cudaSuccess &&
        r2 == cudaDriverEntryPointSuccess) {
      wr = (MemOp64Fn)p;
      wt = (MemOp64Fn)q;
    }
  });
  if (!wr || !wt) return false;
  const int G = h->cfg.split_world, me = h->cfg.split_rank;
  for (int g = 0; g < G; ++g)
    if (g != me && wr((CUstream)st, (CUdeviceptr)(h->peer_bases[g] + 8 * me), epoch, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
      return false;
  for (int g = 0; g < G; ++g)
    if (g != me && wt((CUstream)st, (CUdeviceptr)(h->peer_bases[me] + 8 * g), epoch, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return false;
  return true;
}

static stca_status forward_body(stca_handle *h, const void *xt, int64_t Nt, const int64_t *tgt_off, int64_t B,
                                float *out_Z, float *out_z, cudaStream_t st) {
  stca_status s = STCA_OK;
  const int d = h->cfg.d, hh = h->cfg.h, M = h->cfg.M, es = h->es;
  const int64_t NQ = Nt * hh;  // query rows (target, head)
  const int64_t ldo = (int64_t)(M + 1) * d;

  // inputs: x_t into block 0 of the concatenation buffer [x_t | o1 | ... | oM] (R10)
  const void *xtd = xt;
  const bool host_xt = !is_device_ptr(xt);
  if (host_xt) {  // on the copy stream, behind this step's history upload (the H2D engine is FIFO)
    s = ensure_copy_stream(h, st);
    if (s != STCA_OK) return s;
    void *const old = h->xtin.p;
    CU(h->xtin.ensure((size_t)Nt * d * es, st));
    if (h->xtin.p != old) CU(cudaEventRecord(h->ev_xtin_free, st));
    CU(cudaStreamWaitEvent(h->copy_st, h->ev_xtin_free, 0));  // the previous forward has read x_t
    CU(cudaMemcpyAsync(h->xtin.p, xt, (size_t)Nt * d * es, cudaMemcpyHostToDevice, h->copy_st));
    CU(cudaEventRecord(h->ev_xt_in, h->copy_st));
    CU(cudaStreamWaitEvent(st, h->ev_xt_in, 0));
    xtd = h->xtin.p;
  }
  float *Zd = out_Z, *zd = out_z;
  const bool Z_host = !is_device_ptr(out_Z), z_host = out_z && !is_device_ptr(out_z);
  if (Z_host) {
    CU(h->Zout.ensure((size_t)Nt * M * d * 4, st));
    Zd = h->Zout.as<float>();
  }
  if (z_host) {
    CU(h->zout.ensure((size_t)Nt * d * 4, st));
    zd = h->zout.as<float>();
  }
  CU(h->ocat.ensure((size_t)Nt * ldo * es, st));
  CU(h->q.ensure((size_t)Nt * d * es, st));
  CU(h->c.ensure((size_t)Nt * d * es, st));
  CU(h->U.ensure((size_t)NQ * d * es, st));
  CU(h->Y.ensure((size_t)NQ * d * es, st));
  CU(stca::copy_rows_strided(xtd, (int64_t)d * es, h->ocat.p, ldo * es, Nt, d * es, st));
  if (host_xt) CU(cudaEventRecord(h->ev_xtin_free, st));

  // attention plan (host, exact): items in LPT order, partial rows for multi-chunk requests
  const bool tc_attn = h->bf16 && stca::tc_attention_supported(d);
  // d = 256 / 512: the single-CTA M = 64 kernel (tc_attn_wide.cu).  The CTA-pair kernel (tc_attn_pair.cu,
  // M = 128 per pair at full MMA rate) measured slower -- its SS A operand (U) is re-read from shared
  // memory for every 64-key tile, so it is shared-memory-bandwidth bound; it is built only
  // for A/B runs (-DSTCA_PAIR_ATTN).
#ifdef STCA_PAIR_ATTN
  const bool tc_wide = h->bf16 && stca::tc_attention_pair_supported(d);
  const int wide_qtile = 128;
#else
  const bool tc_wide = h->bf16 && stca::tc_attention_wide_supported(d);
  const int wide_qtile = 64;
#endif
  // A request with at most 64 query rows (m_b h) takes the transposed kernel (keys = MMA rows), which
  // does not pad it to a 128-row query tile.  The choice is PER REQUEST (its items are moved behind
  // the others and launched separately), so a request's arithmetic never depends on its batch
  // (RLB invariance, P10).  STCA_NO_NARROW=1 disables it (A/B runs).
  static const bool no_narrow = getenv("STCA_NO_NARROW") && atoi(getenv("STCA_NO_NARROW")) != 0;
  // a request with m_b h <= 32 takes the 32-column instantiation (also per request); STCA_NO_NARROW32=1
  // sends it to the 64-column one (A/B runs)
  static const bool no_narrow32 = getenv("STCA_NO_NARROW32") && atoi(getenv("STCA_NO_NARROW32")) != 0;
  const bool tc_narrow = tc_attn && !no_narrow;
  const int qtile = tc_attn ? 128 : tc_wide ? wide_qtile : 16;
  std::vector<int64_t> it6;
  int64_t nit = stca_plan_attention(h->len.data(), tgt_off, B, hh, qtile, (int32_t)h->chunk_cap, nullptr, 0);
  it6.resize((size_t)std::max<int64_t>(nit, 1) * 6);
  stca_plan_attention(h->len.data(), tgt_off, B, hh, qtile, (int32_t)h->chunk_cap, it6.data(), nit);
  std::vector<int64_t> part_base(B, -1);
  std::vector<stca::MergeItem> mi;
  int64_t part_rows = 0;
  int max_rows = 0, max_chunks = 0;
  const int G = h->cfg.split_world, grank = h->cfg.split_rank;
  for (int64_t b = 0; b < B; ++b) {
    const int64_t rows = (tgt_off[b + 1] - tgt_off[b]) * hh;
    const int32_t nc = stca_plan_chunks(h->len[b], (int32_t)h->chunk_cap, nullptr);
    if (rows == 0 || (nc <= 1 && G == 1)) continue;  // split-history: every request goes through the merge
    part_base[b] = part_rows;
    mi.push_back({tgt_off[b] * hh, part_rows, (int32_t)rows, nc});
    part_rows += rows * nc;
    max_rows = std::max<int>(max_rows, (int)rows);
    max_chunks = std::max<int>(max_chunks, (int)nc);
  }
  std::vector<stca::AttnItem> items, items_nar[2];  // narrow: [0] 64 query columns, [1] 32
  items.reserve((size_t)nit);
  for (int64_t i = 0; i < nit; ++i) {
    const int64_t *o = &it6[6 * i];
    const int64_t b = o[0];
    if (G > 1) {  // split-history: only the chunks this rank owns (floor(c G / C) == rank)
      const int32_t nc = stca_plan_chunks(h->len[b], (int32_t)h->chunk_cap, nullptr);
      if ((o[5] * G) / nc != grank) continue;
    }
    const int64_t brows = (tgt_off[b + 1] - tgt_off[b]) * hh;
    const bool nar = tc_narrow && stca::tc_attention_narrow_supported(d, (int)std::min<int64_t>(brows, 1 << 30));
    std::vector<stca::AttnItem> &dst = nar ? items_nar[brows <= 32 && !no_narrow32] : items;
    dst.emplace_back();
    stca::AttnItem &a = dst.back();
    a.qrow0 = o[1];
    a.nq = (int32_t)o[2];
    a.key0 = h->coff[b] + (o[3] - h->own0[b]);
    a.klen = (int32_t)o[4];
    a.chunk = (int32_t)o[5];
    a.pad = 0;
    a.part_row = part_base[b] < 0 ? -1 : part_base[b] + o[5] * (tgt_off[b + 1] - tgt_off[b]) * hh + (o[1] - tgt_off[b] * hh);
  }
  const bool stdf = h->attn_form == STCA_FORM_STANDARD;
  if (stdf) {  // standard form: one item per (request, head) over the request's K^r / V^r, all on the narrow kernel
    if (G > 1) return fail(h, STCA_ERR_UNSUPPORTED, "the standard attention form has no split-history mode");
    items.clear();
    items_nar[0].clear();
    items_nar[1].clear();
    mi.clear();
    part_rows = 0;
    for (int64_t b = 0; b < B; ++b) {
      const int64_t mb = tgt_off[b + 1] - tgt_off[b];
      if (mb == 0) continue;
      if (mb > 64)
        return fail(h, STCA_ERR_UNSUPPORTED, "the standard attention form takes <= 64 targets per request (request %lld "
                    "has %lld)", (long long)b, (long long)mb);
      for (int r = 0; r < hh; ++r) {
        stca::AttnItem a{};
        a.qrow0 = tgt_off[b];
        a.nq = (int32_t)mb;
        a.key0 = h->coff[b];
        a.klen = (int32_t)h->len[b];
        a.chunk = 0;
        a.pad = r;
        a.part_row = -1;
        items_nar[mb <= 32 && !no_narrow32].push_back(a);
      }
    }
  }
  const int64_t nit_reg = (int64_t)items.size();
  const int64_t nit_nar[2] = {(int64_t)items_nar[0].size(), (int64_t)items_nar[1].size()};
  const int64_t nar_first[2] = {nit_reg, nit_reg + nit_nar[0]};
  // [128-row kernel items | narrow 64-column items | narrow 32-column items]
  for (int k = 0; k < 2; ++k) items.insert(items.end(), items_nar[k].begin(), items_nar[k].end());
  nit = (int64_t)items.size();
  // persistent d = 128 attention: LPT bins of work items over the SMs (cost = key tiles + 2 for the
  // item's prologue / epilogue), CTA c runs cta_items[cta_off[c] .. cta_off[c+1]) in LPT order
  int n_ctas = 0;
  std::vector<int32_t> ctal;  // cta_off [n_ctas + 1] | cta_items [nit]
  if (tc_attn && nit_reg > 0) {
    n_ctas = (int)std::min<int64_t>(stca::tc_attention_ctas(), nit_reg);
    std::vector<int64_t> cost((size_t)nit_reg);
    for (int64_t i = 0; i < nit_reg; ++i) cost[i] = (items[i].klen + 127) / 128 + 2;
    std::vector<int32_t> bin((size_t)nit_reg);
    stca_plan_persistent(cost.data(), nit_reg, n_ctas, ctal_resize(ctal, n_ctas, nit_reg), bin.data());
  }
  // persistent narrow attention: its own LPT lists appended to ctal (indices relative to its items)
  int n_ctas_nar[2] = {0, 0};
  size_t nar_at[2] = {0, 0};
  for (int k = 0; k < 2; ++k) {
    nar_at[k] = ctal.size();
    if (nit_nar[k] == 0) continue;
    n_ctas_nar[k] = (int)std::min<int64_t>(stca::tc_attention_ctas(), nit_nar[k]);
    std::vector<int64_t> cost((size_t)nit_nar[k]);
    for (int64_t i = 0; i < nit_nar[k]; ++i) cost[i] = (items[nar_first[k] + i].klen + 127) / 128 + 2;
    std::vector<int32_t> bin((size_t)nit_nar[k]), v;
    stca_plan_persistent(cost.data(), nit_nar[k], n_ctas_nar[k], ctal_resize(v, n_ctas_nar[k], nit_nar[k]), bin.data());
    ctal.insert(ctal.end(), v.begin(), v.end());
  }
  // the plan [items | merge items | CTA lists], 256-byte aligned sections, in one upload
  const size_t items_bytes = items.size() * sizeof(stca::AttnItem), mi_bytes = mi.size() * sizeof(stca::MergeItem);
  const size_t ctal_bytes = ctal.size() * sizeof(int32_t);
  const size_t mi_at = (items_bytes + 255) / 256 * 256, ctal_at = mi_at + (mi_bytes + 255) / 256 * 256;
  {
    std::vector<uint8_t> pl(ctal_at + ctal_bytes);
    if (items_bytes) memcpy(pl.data(), items.data(), items_bytes);
    if (mi_bytes) memcpy(pl.data() + mi_at, mi.data(), mi_bytes);
    if (ctal_bytes) memcpy(pl.data() + ctal_at, ctal.data(), ctal_bytes);
    s = upload_plan(h, pl.data(), pl.size(), h->plan, st);
    if (s != STCA_OK) return s;
  }
  stca::AttnItem *d_items = h->plan.as<stca::AttnItem>();
  stca::MergeItem *d_mitems = reinterpret_cast<stca::MergeItem *>(h->plan.as<uint8_t>() + mi_at);
  int32_t *d_ctal = reinterpret_cast<int32_t *>(h->plan.as<uint8_t>() + ctal_at);
  const size_t part_bytes = (size_t)part_rows * stca::part_row_bytes(d, es);
  const bool peer = G > 1 && h->peer_on;
  if (G > 1 && !peer && !h->cfg.exchange)
    return fail(h, STCA_ERR_INVALID_ARG, "split-history needs an exchange callback or attached peer buffers");
  if (peer && (int64_t)part_bytes > h->peer_cap)
    return fail(h, STCA_ERR_INVALID_ARG, "the partials (%zu bytes) exceed the peer buffer slot (%lld bytes)", part_bytes,
                (long long)h->peer_cap);
  if (part_rows && !peer) CU(h->part.ensure(part_bytes, st));
  if (G > 1 && part_rows && !peer) CU(h->partg.ensure(part_bytes * G, st));
  const uint64_t *const flags_ready = peer ? (const uint64_t *)h->peer_buf : nullptr;

  // target side: at d = 128 every layer boundary is ONE fused kernel (tc_chain.cu: o(i) -> Z, ocat;
  // c = [..] W_C; q = SwiGLUFFN(c); U = q W_QK), otherwise separate tcgen05 GEMMs / CUDA-core kernels
#ifdef STCA_NO_CHAIN  // A/B builds only: the separate-GEMM target side
  const bool chain = false;
#else
  const bool chain = h->bf16 && stca::tc_chain_supported(d, hh, h->cfg.r * d);
#endif
  if (stdf && !chain) return fail(h, STCA_ERR_UNSUPPORTED, "the standard attention form runs with the fused target side");
  if (stdf) CU(h->kvbuf.ensure((size_t)std::max<int64_t>(h->T2, 1) * hh * d * es, st));
  auto chain_base = [&](int mode) {
    stca::TcChain c;
    c.mode = mode;
    c.M = M;
    c.h = hh;
    c.rd = h->cfg.r * d;
    c.Nt = Nt;
    c.ocat = h->ocat.p;
    c.U = h->U.p;
    c.eps = h->cfg.ln_eps;
    return c;
  };
  // a2: q(1) = LN(SwiGLUFFN(1)(x_t)), Eq.(3)
  LayerW &L1 = h->L[0];
  if (chain) {  // ... and a3 of layer 1
    stca::TcChain c = chain_base(0);
    c.W1t = L1.tc.W1q;
    c.Wot = L1.tc.Woq;
    c.WQKt = stdf ? h->std_q[0].WQK : L1.tc.WQK;
    c.g = L1.gq;
    c.b = L1.bq;
    cudaEvent_t pa = h->prof_target ? prof_begin(h, st) : nullptr;
    CU(stca::tc_chain(c, st));
    prof_end(h, STCA_PH_TARGET, pa, st);
  } else {
    s = ffn_rows(h, h->ocat.p, ldo, Nt, L1.W1q, L1.Woq, &L1.tc, 1, L1.gq, L1.bq, h->q.p, d, nullptr, 0, st);
    if (s != STCA_OK) return s;
  }
  for (int i = 1; i <= M; ++i) {
    LayerW &Ly = h->L[i - 1];
    const void *Xt = (const uint8_t *)h->xt_cache.p + (size_t)(i - 1) * h->T2 * d * es;
    // a3: U = q W_QK (all heads; pre-scaled by log2(e)/sqrt(d_h)) -> [Nt h x d] (fused: by the previous chain)
    if (!chain) {
      s = gemm(h, h->q.p, d, Ly.WQK, Ly.tc.WQK, (int64_t)hh * d, h->U.p, (int64_t)hh * d, nullptr, 0, Nt, hh * d, d, st);
      if (s != STCA_OK) return s;
    }
    // a4: ragged single-query attention per request, reordered form Eq.(13)
    float *part_i = h->part.as<float>();
    uint64_t epoch = 0;
    if (peer) {  // this layer's slot of the exchange buffer (the peers read it two layers ago: see below)
      epoch = ++h->epoch;
      part_i = (float *)((uint8_t *)h->peer_buf + 4096 + (size_t)(epoch & 1) * h->peer_cap);
    }
    cudaEvent_t pa = prof_begin(h, st);
    for (int rep = 0; rep < h->reps_attn; ++rep) {  // idempotent (STCA_PROF_TWICE_ATTENTION)
    if (stdf) {  // standard form, Eq.(12): [K^r | V^r | 0] = X~ [W_K^r | W_V^r | 0] for every head, then attention
      if (rep == 0) {
        cudaEvent_t pk = h->prof_target ? prof_begin(h, st) : nullptr;
        CU(stca::tc_gemm(Xt, d, h->std_kv[i - 1].WQK, h->T2, hh * d, d, h->kvbuf.p, (int64_t)hh * d, nullptr, 0, st));
        prof_end(h, STCA_PH_TARGET, pk, st);
      }
      for (int k = 0; k < 2; ++k)
        if (nit_nar[k] > 0)
          CU(stca::tc_attention_narrow(h->U.p, NQ, h->kvbuf.p, h->T2, d_items + nar_first[k], d_ctal + nar_at[k],
                                       d_ctal + nar_at[k] + n_ctas_nar[k] + 1, n_ctas_nar[k], h->Y.p, part_i, st, hh,
                                       k ? 32 : 64));
    } else if (tc_attn) {
      for (int k = 0; k < 2; ++k)
        if (nit_nar[k] > 0)
          CU(stca::tc_attention_narrow(h->U.p, NQ, Xt, h->T2, d_items + nar_first[k], d_ctal + nar_at[k],
                                       d_ctal + nar_at[k] + n_ctas_nar[k] + 1, n_ctas_nar[k], h->Y.p, part_i, st, 1,
                                       k ? 32 : 64));
      if (nit_reg > 0)
        CU(stca::tc_attention(h->U.p, NQ, Xt, h->T2, d_items, d_ctal,
                            d_ctal + n_ctas + 1, n_ctas, d, h->Y.p, part_i, st));
    } else if (tc_wide) {
#ifdef STCA_PAIR_ATTN
      CU(stca::tc_attention_pair(h->U.p, NQ, Xt, h->T2, d_items, nit, d, h->Y.p,
                                 part_i, st));
#else
      CU(stca::tc_attention_wide(h->U.p, NQ, Xt, h->T2, d_items, nit, d, h->Y.p,
                                 part_i, st));
#endif
    } else {
      CU(stca::cc_attention(h->bf16, h->U.p, Xt, d_items, nit, d, h->Y.p, part_i, st));
    }
    }
    prof_end(h, STCA_PH_ATTENTION, pa, st);
    const float *merged_from = part_i;
    // split-history over peer memory: one 1-thread kernel publishes this layer's epoch and waits for every
    // peer's, then the merge reads each chunk in place.  Slot reuse needs no second flag: this rank overwrites slot (e & 1)
    // in layer e + 2 only after its merge of e + 1 saw every peer's epoch e + 1, which a peer publishes
    // only after its own merge of e (the one reading this slot) has completed (stream order + PDL waits).
    stca::PeerMerge pmg{};
    if (peer) {
      pmg.slots = (const uint8_t *const *)(h->peer_tab + (epoch & 1) * G);
      pmg.ready_remote = (uint64_t *const *)(h->peer_tab + 2 * G);
      pmg.ready_local = flags_ready;
      pmg.me = grank;
      pmg.epoch = epoch;
    } else if (G > 1 && part_rows) {  // split-history exchange: all-gather every rank's partials (one step per layer)
      if (h->cfg.exchange(h->cfg.exchange_ctx, h->part.p, h->partg.p, part_bytes, (void *)st) != 0)
        return fail(h, STCA_ERR_COMM, "split-history exchange failed at layer %d", i);
      merged_from = h->partg.as<float>();
    }
    if (h->cap_layer == i) {  // stage-isolated test hook: this layer's U (a3 output) and Y (a4 output)
      CU(cudaMemcpyAsync(h->cap_U, h->U.p, (size_t)NQ * d * es, cudaMemcpyDeviceToDevice, st));
    }
    if (h->save_act)  // stca_backward: U of layer i (slot 2 (i - 1))
      CU(cudaMemcpyAsync(h->act.as<uint8_t>() + (size_t)2 * (i - 1) * NQ * d * es, h->U.p, (size_t)NQ * d * es,
                         cudaMemcpyDeviceToDevice, st));
    pa = prof_begin(h, st);
    if (peer) {  // publish this layer's epoch to every peer, then wait (in the stream) for every peer's
      if (!peer_exchange_memops(h, epoch, st)) CU(stca::peer_exchange(pmg, G, st));
    }
    CU(stca::merge_partials(h->bf16, d_mitems, (int64_t)mi.size(), max_rows, max_chunks, merged_from,
                            peer ? &pmg : nullptr, d, G, (int64_t)part_bytes, h->Y.p, st));
    if (!mi.empty()) prof_end(h, STCA_PH_MERGE, pa, st);
    else if (pa) h->prof_pool.push_back(pa);
    if (h->cap_layer == i) {
      CU(cudaMemcpyAsync(h->cap_Y, h->Y.p, (size_t)NQ * d * es, cudaMemcpyDeviceToDevice, st));
      h->cap_layer = 0;
    }
    if (h->save_act)  // ... and its attention output Y (slot 2 (i - 1) + 1)
      CU(cudaMemcpyAsync(h->act.as<uint8_t>() + (size_t)(2 * (i - 1) + 1) * NQ * d * es, h->Y.p, (size_t)NQ * d * es,
                         cudaMemcpyDeviceToDevice, st));
    if (chain) {  // a5 (+ a6, a3 of layer i + 1; or a7 after the last layer) as one kernel
      stca::TcChain c = chain_base(i < M ? 1 : 2);
      c.Y = h->Y.p;
      c.ocat_out = (uint8_t *)h->ocat.p + (size_t)i * d * es;
      c.Z = Zd + (size_t)(i - 1) * d;
      c.ldz = (int64_t)M * d;
      c.WVOt = stdf ? h->std_q[i - 1].WVO : Ly.tc.WVO;
      if (i < M) {
        LayerW &Ln = h->L[i];
        c.kc = i + 1;
        c.WCt = Ln.tc.WC;
        c.W1t = Ln.tc.W1q;
        c.Wot = Ln.tc.Woq;
        c.WQKt = stdf ? h->std_q[i].WQK : Ln.tc.WQK;
      } else if (zd) {
        c.kc = M + 1;
        c.WCt = h->tcz.WC;
        c.W1t = h->tcz.W1h;
        c.Wot = h->tcz.Woh;
        c.zout = zd;
      }
      cudaEvent_t pa = h->prof_target ? prof_begin(h, st) : nullptr;
      CU(stca::tc_chain(c, st));
      prof_end(h, STCA_PH_TARGET, pa, st);
      continue;
    }
    // a5: o(i) = [Y_r]_r W_VO -> out_Z[:, i] (fp32) and block i of the concatenation (storage)
    s = gemm(h, h->Y.p, (int64_t)hh * d, Ly.WVO, Ly.tc.WVO, d, (uint8_t *)h->ocat.p + (size_t)i * d * es, ldo,
             Zd + (size_t)(i - 1) * d, (int64_t)M * d, Nt, d, hh * d, st);
    if (s != STCA_OK) return s;
    // a6: q(i+1) = SwiGLUFFN(i+1)([o(1)..o(i) | x_t] W_C(i+1)), Eq.(7)
    if (i < M) {
      LayerW &Ln = h->L[i];
      s = gemm(h, h->ocat.p, ldo, Ln.WC, Ln.tc.WC, d, h->c.p, d, nullptr, 0, Nt, d, (i + 1) * d, st);
      if (s != STCA_OK) return s;
      s = ffn_rows(h, h->c.p, d, Nt, Ln.W1q, Ln.Woq, &Ln.tc, 1, nullptr, nullptr, h->q.p, d, nullptr, 0, st);
      if (s != STCA_OK) return s;
    }
  }
  // a7: z = SwiGLUFFN_Z([o(1)..o(M) | x_t] W_Z), Eq.(9) (fused: by the last chain)
  if (zd && !chain) {
    s = gemm(h, h->ocat.p, ldo, h->WZ, h->tcz.WC, d, h->c.p, d, nullptr, 0, Nt, d, (M + 1) * d, st);
    if (s != STCA_OK) return s;
    s = ffn_rows(h, h->c.p, d, Nt, h->W1z, h->Woz, &h->tcz, 0, nullptr, nullptr, nullptr, 0, zd, d, st);
    if (s != STCA_OK) return s;
  }
  if (Z_host) CU(cudaMemcpyAsync(out_Z, Zd, (size_t)Nt * M * d * 4, cudaMemcpyDeviceToHost, st));
  if (z_host) CU(cudaMemcpyAsync(out_z, zd, (size_t)Nt * d * 4, cudaMemcpyDeviceToHost, st));
  // host outputs: asynchronous like every other result (complete once `stream` reaches this point)
  CU(cudaGetLastError());
  return STCA_OK;
}

// ===========================================================================
// stca_profile: per-phase CUDA-event regions on the launching stream
// ===========================================================================
extern "C" stca_status stca_profile(stca_handle *h, int32_t enable) {
  if (!h) return STCA_ERR_INVALID_ARG;
  h->prof = (enable & STCA_PROF_EVENTS) != 0;
  h->prof_target = h->prof && (enable & STCA_PROF_EVENTS_TARGET) != 0;
  h->reps_attn = (enable & STCA_PROF_TWICE_ATTENTION) ? 2 : 1;
  h->reps_proj = (enable & STCA_PROF_TWICE_PROJECT) ? 2 : 1;
  return STCA_OK;
}

extern "C" stca_status stca_profile_read(stca_handle *h, double *ms, int64_t *count) {
  if (!h || !ms || !count) return STCA_ERR_INVALID_ARG;
  for (int p = 0; p < STCA_PH_N; ++p) {
    ms[p] = 0.0;
    count[p] = 0;
  }
  CU(cudaSetDevice(h->cfg.device));
  for (ProfRegion &r : h->prof_open) {
    CU(cudaEventSynchronize(r.b));
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.phase] += t;
    count[r.phase] += 1;
    h->prof_pool.push_back(r.a);
    h->prof_pool.push_back(r.b);
  }
  h->prof_open.clear();
  return STCA_OK;
}

// Stage-isolated test hook (not part of include/stca.h): during the next stca_forward, copy layer
// `layer`'s reordered queries U [Nt h x d] (a3, pre-scaled by log2(e)/sqrt(d_h)) and the attention
// output Y [Nt h x d] (a4 after the split-K fold) in the storage type into the caller's DEVICE
// buffers, so a test can re-evaluate the softmax in f64 from the GPU's own bf16 operands.
extern "C" stca_status stca_debug_capture(stca_handle *h, int32_t layer, void *U_out, void *Y_out) {
  if (!h || !U_out || !Y_out || layer < 1 || layer > h->cfg.M) return STCA_ERR_INVALID_ARG;
  h->cap_layer = layer;
  h->cap_U = U_out;
  h->cap_Y = Y_out;
  return STCA_OK;
}

// ===========================================================================
// NEXT-1 (partial): backward of one layer's attention with request-level gradient aggregation
// ===========================================================================
// attention-backward work items: (request, block of <= 64 query rows) over ALL of the request's kept keys
static std::vector<stca::AttnItem> bwd_items(const stca_handle *h, const int64_t *tgt_off, int64_t B) {
  const int hh = h->cfg.h;
  std::vector<stca::AttnItem> items;
  for (int64_t b = 0; b < B; ++b) {
    const int64_t rows = (tgt_off[b + 1] - tgt_off[b]) * hh;
    const int64_t nqb = (rows + 63) / 64;
    for (int64_t qb = 0; qb < nqb; ++qb) {
      stca::AttnItem a{};
      a.qrow0 = tgt_off[b] * hh + 64 * qb;
      a.nq = (int32_t)std::min<int64_t>(64, rows - 64 * qb);
      a.key0 = h->coff[b];
      a.klen = (int32_t)h->len[b];
      a.chunk = 0;
      a.part_row = nqb > 1 ? 1 : 0;  // several items add into the request's dX~ rows
      items.push_back(a);
    }
  }
  return items;
}

extern "C" stca_status stca_attention_backward(stca_handle *h, int32_t layer, const void *U, const float *dY,
                                               const int64_t *tgt_off, int64_t B, float *dXt, float *dU,
                                               void *stream) {
  if (!h) return STCA_ERR_INVALID_ARG;
  if (h->sticky) return fail(h, STCA_ERR_CUDA, "handle is in a sticky CUDA error state: %s", h->err.c_str());
  if (h->B < 0) return fail(h, STCA_ERR_STATE, "stca_attention_backward before stca_project_history");
  if (B != h->B) return fail(h, STCA_ERR_STATE, "B=%lld differs from the projected B=%lld", (long long)B, (long long)h->B);
  if (!h->bf16 || h->cfg.d != 128)
    return fail(h, STCA_ERR_UNSUPPORTED, "the attention backward runs on the bf16 path with d = 128 (d=%d)", h->cfg.d);
  if (h->cfg.split_world > 1) return fail(h, STCA_ERR_UNSUPPORTED, "no attention backward in split-history mode");
  if (layer < 1 || layer > h->cfg.M) return fail(h, STCA_ERR_INVALID_ARG, "layer %d outside 1..%d", layer, h->cfg.M);
  if (!tgt_off) return fail(h, STCA_ERR_INVALID_ARG, "tgt_off is NULL");
  const int64_t Nt = tgt_off[B];
  int64_t badi = -1;
  stca_status s = check_offsets(tgt_off, B, Nt, false, &badi);
  if (s != STCA_OK) return fail(h, s, "tgt_off invalid at request %lld", (long long)badi);
  if (Nt > 0 && (!U || !dY || !dU)) return fail(h, STCA_ERR_INVALID_ARG, "NULL U / dY / dU");
  if (!dXt) return fail(h, STCA_ERR_INVALID_ARG, "dXt is NULL");
  CU(cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  const int d = h->cfg.d, hh = h->cfg.h;
  const int64_t NQ = Nt * hh;
  std::vector<stca::AttnItem> items = bwd_items(h, tgt_off, B);
  // dX~ rows of requests without targets (and the sums of multi-block requests) start from zero
  CU(cudaMemsetAsync(dXt, 0, (size_t)h->T2 * d * sizeof(float), st));
  if (items.empty()) return STCA_OK;
  s = upload_plan(h, items.data(), items.size() * sizeof(stca::AttnItem), h->seg, st);
  if (s != STCA_OK) return s;
  const void *Xt = (const uint8_t *)h->xt_cache.p + (size_t)(layer - 1) * h->T2 * d * h->es;
  CU(stca::tc_attention_bwd(U, NQ, Xt, h->T2, h->seg.as<stca::AttnItem>(), (int64_t)items.size(), dY, dXt, dU, st));
  return STCA_OK;
}

extern "C" stca_status stca_history_backward(stca_handle *h, int32_t layer, const void *X, int64_t rows,
                                             const float *dXt, float *dX, float *dWu, float *dWv, float *dWo,
                                             float *dgamma, float *dbeta, void *stream) {
  if (!h) return STCA_ERR_INVALID_ARG;
  if (h->sticky) return fail(h, STCA_ERR_CUDA, "handle is in a sticky CUDA error state: %s", h->err.c_str());
  if (h->B < 0) return fail(h, STCA_ERR_STATE, "stca_history_backward before stca_project_history");
  if (!h->bf16) return fail(h, STCA_ERR_UNSUPPORTED, "the history backward runs on the bf16 path");
  if (h->sess_on) return fail(h, STCA_ERR_UNSUPPORTED, "no history backward over a session cache");
  if (layer < 1 || layer > h->cfg.M) return fail(h, STCA_ERR_INVALID_ARG, "layer %d outside 1..%d", layer, h->cfg.M);
  if (rows != h->T2)
    return fail(h, STCA_ERR_SHAPE, "X has %lld rows, the projection kept %lld", (long long)rows, (long long)h->T2);
  if (rows > 0 && (!X || !dXt || !dX)) return fail(h, STCA_ERR_INVALID_ARG, "NULL X / dXt / dX");
  if (!dWu || !dWv || !dWo || !dgamma || !dbeta) return fail(h, STCA_ERR_INVALID_ARG, "NULL weight gradient");
  CU(cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  const int d = h->cfg.d, rd = h->cfg.r * d;
  const int64_t R = std::min<int64_t>(std::max<int64_t>(rows, 1), STCA_BWD_ROWS);
  CU(h->bwd_scratch.ensure(stca::hist_bwd_scratch_bytes(d, rd, R), st));
  LayerW &Ly = h->L[layer - 1];
  CU(stca::hist_bwd(&h->blas, (const bf16 *)X, rows, d, rd, (const bf16 *)Ly.W1cat,
                    (const bf16 *)Ly.Woh, Ly.tc.W1h, Ly.tc.Woh, Ly.gh, h->cfg.ln_eps, dXt, dX, dWu, dWv, dWo, dgamma, dbeta,
                    h->bwd_scratch.p, R, st));
  return STCA_OK;
}

// ===========================================================================
// NEXT-1: backward of the whole stack (forward with saved U / Y, then target side in reverse order with
// each layer's attention and history backward in between)
// ===========================================================================
namespace {
struct BwdCtx {
  stca_handle *h;
  const void *X;
  int64_t rows, NQ, nit;
  const stca::AttnItem *items;
  float *dX;
  float *gWu[STCA_MAX_LAYERS], *gWv[STCA_MAX_LAYERS], *gWo[STCA_MAX_LAYERS], *gg[STCA_MAX_LAYERS], *gb[STCA_MAX_LAYERS];
  cudaStream_t st;
};
}  // namespace

static cudaError_t bwd_attn_hist(void *ctx, int layer, const float *dY, float *dU) {
  BwdCtx &c = *(BwdCtx *)ctx;
  stca_handle *h = c.h;
  const int d = h->cfg.d, rd = h->cfg.r * d, L = layer - 1;
  float *dXt = h->dxt_buf.as<float>();
  cudaError_t e = cudaMemsetAsync(dXt, 0, (size_t)h->T2 * d * 4, c.st);
  if (e != cudaSuccess) return e;
  const void *U = h->act.as<uint8_t>() + (size_t)2 * L * c.NQ * d * h->es;
  const void *Xt = (const uint8_t *)h->xt_cache.p + (size_t)L * h->T2 * d * h->es;
  if (c.nit > 0 && (e = stca::tc_attention_bwd(U, c.NQ, Xt, h->T2, c.items, c.nit, dY, dXt, dU, c.st)) != cudaSuccess)
    return e;
  const int64_t R = std::min<int64_t>(std::max<int64_t>(c.rows, 1), STCA_BWD_ROWS);
  LayerW &Ly = h->L[L];
  return stca::hist_bwd(&h->blas, (const bf16 *)c.X, c.rows, d, rd, (const bf16 *)Ly.W1cat,
                        (const bf16 *)Ly.Woh, Ly.tc.W1h, Ly.tc.Woh, Ly.gh, h->cfg.ln_eps, dXt, c.dX, c.gWu[L], c.gWv[L], c.gWo[L], c.gg[L],
                        c.gb[L], h->bwd_scratch.p, R, c.st);
}

extern "C" stca_status stca_backward(stca_handle *h, const void *xt, int64_t Nt, const int64_t *tgt_off, int64_t B,
                                     const void *X, int64_t rows, const float *dZ, const float *dz,
                                     const stca_grad *grads, int32_t n_grads, float *dX, float *dxt, float *out_Z,
                                     void *stream) {
  if (!h) return STCA_ERR_INVALID_ARG;
  if (h->sticky) return fail(h, STCA_ERR_CUDA, "handle is in a sticky CUDA error state: %s", h->err.c_str());
  if (h->B < 0) return fail(h, STCA_ERR_STATE, "stca_backward before stca_project_history");
  if (B != h->B) return fail(h, STCA_ERR_STATE, "B=%lld differs from the projected B=%lld", (long long)B, (long long)h->B);
  if (!h->bf16 || h->cfg.d != 128)
    return fail(h, STCA_ERR_UNSUPPORTED, "the backward runs on the bf16 path with d = 128 (d=%d)", h->cfg.d);
  if (h->cfg.split_world > 1) return fail(h, STCA_ERR_UNSUPPORTED, "no backward in split-history mode");
  if (h->sess_on) return fail(h, STCA_ERR_UNSUPPORTED, "no backward over a session cache");
  if (!tgt_off) return fail(h, STCA_ERR_INVALID_ARG, "tgt_off is NULL");
  int64_t badi = -1;
  stca_status s = check_offsets(tgt_off, B, Nt, false, &badi);
  if (s != STCA_OK) return fail(h, s, "tgt_off invalid at request %lld", (long long)badi);
  if (rows != h->T2)
    return fail(h, STCA_ERR_SHAPE, "X has %lld rows, the projection kept %lld", (long long)rows, (long long)h->T2);
  if (n_grads < 0 || (n_grads > 0 && !grads)) return fail(h, STCA_ERR_INVALID_ARG, "bad gradient list");
  const int d = h->cfg.d, hh = h->cfg.h, r = h->cfg.r, M = h->cfg.M, rd = r * d;
  const bool wz = h->cfg.with_z != 0;
  // every device argument must be device memory (the backward keeps no host staging)
  auto dev = [&](const void *p, const char *what) -> stca_status {
    if (p && !is_device_ptr(p)) return fail(h, STCA_ERR_INVALID_ARG, "%s must be device memory", what);
    return STCA_OK;
  };
  if (Nt > 0 && (!xt || !dZ)) return fail(h, STCA_ERR_INVALID_ARG, "NULL x_t / dZ");
  if (rows > 0 && !X) return fail(h, STCA_ERR_INVALID_ARG, "NULL X");
  if (dz && !wz) return fail(h, STCA_ERR_INVALID_ARG, "dz given but the handle has with_z = 0");
  for (auto pr : {std::make_pair((const void *)xt, "x_t"), std::make_pair((const void *)X, "X"),
                  std::make_pair((const void *)dZ, "dZ"), std::make_pair((const void *)dz, "dz"),
                  std::make_pair((const void *)dX, "dX"), std::make_pair((const void *)dxt, "dxt"),
                  std::make_pair((const void *)out_Z, "out_Z")})
    if ((s = dev(pr.first, pr.second)) != STCA_OK) return s;
  // gradient buffers by role name; roles not asked for accumulate into a sink
  const std::vector<Need> roles = weight_roles(d, r, M, wz);
  std::map<std::string, float *> g;
  for (int32_t i = 0; i < n_grads; ++i) {
    if (!grads[i].name || !grads[i].grad) return fail(h, STCA_ERR_INVALID_ARG, "gradient %d has a NULL name or buffer", i);
    bool known = false;
    for (const Need &n : roles) known |= n.name == grads[i].name;
    if (!known) return fail(h, STCA_ERR_INVALID_ARG, "unknown weight '%s'", grads[i].name);
    if (g.count(grads[i].name)) return fail(h, STCA_ERR_INVALID_ARG, "duplicate gradient '%s'", grads[i].name);
    if ((s = dev(grads[i].grad, grads[i].name)) != STCA_OK) return s;
    g[grads[i].name] = grads[i].grad;
  }
  CU(cudaSetDevice(h->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t NQ = Nt * hh;
  size_t sink = 0;
  for (const Need &n : roles)
    if (!g.count(n.name)) sink += (size_t)(n.rows * n.cols + 63) / 64 * 64;
  CU(h->gsink.ensure(std::max<size_t>(sink, 1) * 4, st));
  {
    float *q = h->gsink.as<float>();
    for (const Need &n : roles)
      if (!g.count(n.name)) {
        g[n.name] = q;
        q += (size_t)(n.rows * n.cols + 63) / 64 * 64;
      }
  }
  for (const Need &n : roles) CU(cudaMemsetAsync(g[n.name], 0, (size_t)n.rows * n.cols * 4, st));
  if (dX && rows > 0) CU(cudaMemsetAsync(dX, 0, (size_t)rows * d * 4, st));
  if (Nt == 0) return STCA_OK;  // no target: every gradient is zero
  // ---- forward, keeping every layer's U and Y ----
  CU(h->act.ensure((size_t)2 * M * NQ * d * h->es, st));
  float *Zd = out_Z;
  if (!Zd) {
    CU(h->Zout.ensure((size_t)Nt * M * d * 4, st));
    Zd = h->Zout.as<float>();
  }
  h->save_act = true;
  s = forward_body(h, xt, Nt, tgt_off, B, Zd, nullptr, st);
  h->save_act = false;
  if (s != STCA_OK) return s;
  // ---- backward ----
  std::vector<stca::AttnItem> items = bwd_items(h, tgt_off, B);
  if (!items.empty()) {
    s = upload_plan(h, items.data(), items.size() * sizeof(stca::AttnItem), h->seg, st);
    if (s != STCA_OK) return s;
  }
  CU(h->dxt_buf.ensure((size_t)std::max<int64_t>(h->T2, 1) * d * 4, st));
  const int64_t R = std::min<int64_t>(std::max<int64_t>(rows, 1), STCA_BWD_ROWS);
  CU(h->bwd_scratch.ensure(stca::hist_bwd_scratch_bytes(d, rd, R), st));
  CU(h->sbwd_scratch.ensure(stca::stack_bwd_scratch_bytes(d, hh, rd, M, Nt), st));
  // dX: the history backward accumulates into it; without a caller buffer it goes to scratch
  float *dXd = dX;
  if (!dXd) {
    CU(h->dxsink.ensure((size_t)std::max<int64_t>(rows, 1) * d * 4, st));
    dXd = h->dxsink.as<float>();
  }
  BwdCtx c{};
  c.h = h;
  c.X = X;
  c.rows = rows;
  c.NQ = NQ;
  c.nit = (int64_t)items.size();
  c.items = h->seg.as<stca::AttnItem>();
  c.dX = dXd;
  c.st = st;
  stca::StackBwd a{};
  a.d = d;
  a.h = hh;
  a.rd = rd;
  a.M = M;
  a.eps = h->cfg.ln_eps;
  a.with_z = wz;
  a.Nt = Nt;
  a.xt = (const bf16 *)xt;
  a.dZ = dZ;
  a.dz = dz;
  for (int i = 1; i <= M; ++i) {
    const std::string p = "L" + std::to_string(i) + ".";
    const int L = i - 1;
    a.Y[L] = (const bf16 *)(h->act.as<uint8_t>() + (size_t)(2 * L + 1) * NQ * d * h->es);
    a.qWu[L] = h->w32[p + "qry.Wu"];
    a.qWv[L] = h->w32[p + "qry.Wv"];
    a.qWo[L] = h->w32[p + "qry.Wo"];
    a.WQ[L] = h->w32[p + "WQ"];
    a.WK[L] = h->w32[p + "WK"];
    a.WV[L] = h->w32[p + "WV"];
    a.WO[L] = h->w32[p + "WO"];
    a.WC[L] = i >= 2 ? h->w32[p + "WC"] : nullptr;
    a.g_qWu[L] = g[p + "qry.Wu"];
    a.g_qWv[L] = g[p + "qry.Wv"];
    a.g_qWo[L] = g[p + "qry.Wo"];
    a.g_WQ[L] = g[p + "WQ"];
    a.g_WK[L] = g[p + "WK"];
    a.g_WV[L] = g[p + "WV"];
    a.g_WO[L] = g[p + "WO"];
    a.g_WC[L] = i >= 2 ? g[p + "WC"] : nullptr;
    c.gWu[L] = g[p + "hist.Wu"];
    c.gWv[L] = g[p + "hist.Wv"];
    c.gWo[L] = g[p + "hist.Wo"];
    c.gg[L] = g[p + "hist.ln_g"];
    c.gb[L] = g[p + "hist.ln_b"];
  }
  a.qg = h->w32["L1.qry.ln_g"];
  a.qb = h->w32["L1.qry.ln_b"];
  a.g_qg = g["L1.qry.ln_g"];
  a.g_qb = g["L1.qry.ln_b"];
  if (wz) {
    a.WZ = h->w32["z.WZ"];
    a.zWu = h->w32["z.Wu"];
    a.zWv = h->w32["z.Wv"];
    a.zWo = h->w32["z.Wo"];
    a.g_WZ = g["z.WZ"];
    a.g_zWu = g["z.Wu"];
    a.g_zWv = g["z.Wv"];
    a.g_zWo = g["z.Wo"];
  }
  a.dxt = dxt;
  a.attn_hist = bwd_attn_hist;
  a.ctx = &c;
  a.scratch = h->sbwd_scratch.p;
  CU(stca::stack_bwd(&h->blas, a, st));
  return STCA_OK;
}

// ===========================================================================
// split-history over peer memory (NVLink / NVSwitch): one exchange buffer per rank, read in place by
// every peer's merge kernel; epoch flags instead of a collective
// ===========================================================================
extern "C" stca_status stca_split_peer_export(stca_handle *h, int64_t capacity_bytes, void **base_out,
                                              void *ipc_handle_out) {
  if (!h || !base_out || capacity_bytes <= 0) return STCA_ERR_INVALID_ARG;
  if (h->cfg.split_world < 2) return fail(h, STCA_ERR_STATE, "peer buffers need split-history mode (split_world >= 2)");
  if (h->peer_buf) return fail(h, STCA_ERR_STATE, "the peer buffer was already exported");
  CU(cudaSetDevice(h->cfg.device));
  const int64_t cap = (capacity_bytes + 4095) / 4096 * 4096;
  void *p = nullptr;
  if (cudaMalloc(&p, (size_t)(4096 + 2 * cap)) != cudaSuccess) {
    cudaGetLastError();
    return fail(h, STCA_ERR_OOM, "peer buffer of %lld bytes", (long long)(4096 + 2 * cap));
  }
  h->peer_buf = p;
  h->peer_cap = cap;
  CU(cudaMemset(p, 0, 4096));  // epoch flags start at 0 (synchronous: before any peer can see the buffer)
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, h->cfg.device));
  memcpy(h->peer_uuid, &prop.uuid, 16);
  CU(cudaMemcpy((uint8_t *)p + 1024, h->peer_uuid, 16, cudaMemcpyHostToDevice));  // read by the peers' attach
  if (ipc_handle_out) CU(cudaIpcGetMemHandle((cudaIpcMemHandle_t *)ipc_handle_out, p));
  *base_out = p;
  return STCA_OK;
}

extern "C" stca_status stca_split_peer_attach(stca_handle *h, void *const *bases) {
  if (!h || !bases) return STCA_ERR_INVALID_ARG;
  const int G = h->cfg.split_world, me = h->cfg.split_rank;
  if (!h->peer_buf) return fail(h, STCA_ERR_STATE, "stca_split_peer_attach before stca_split_peer_export");
  if (bases[me] != h->peer_buf) return fail(h, STCA_ERR_INVALID_ARG, "bases[%d] is not this rank's exported buffer", me);
  std::vector<void *> tab((size_t)3 * G);
  for (int g = 0; g < G; ++g) {
    if (!bases[g]) return fail(h, STCA_ERR_INVALID_ARG, "bases[%d] is NULL", g);
    if (g != me) {  // the exporter wrote its device's UUID at byte 1024 of its buffer
      uint8_t uu[16];
      if (cudaMemcpy(uu, (const uint8_t *)bases[g] + 1024, 16, cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return fail(h, STCA_ERR_INVALID_ARG, "bases[%d] is not readable from this process", g);
      }
      if (memcmp(uu, h->peer_uuid, 16) == 0)
        return fail(h, STCA_ERR_UNSUPPORTED,
                    "peer exchange needs one rank per device (rank %d is on this rank's device): ranks sharing a "
                    "device wait for each other inside their streams and can serialise on its work queues", g);
    }
    uint8_t *b = (uint8_t *)bases[g];
    tab[g] = b + 4096;
    tab[G + g] = b + 4096 + h->peer_cap;
    tab[2 * G + g] = b;  // ready flags of rank g
  }
  CU(cudaSetDevice(h->cfg.device));
  if (!h->peer_tab) CU(cudaMalloc((void **)&h->peer_tab, tab.size() * sizeof(void *)));
  CU(cudaMemcpy(h->peer_tab, tab.data(), tab.size() * sizeof(void *), cudaMemcpyHostToDevice));
  h->peer_bases.assign((uint8_t *const *)bases, (uint8_t *const *)bases + G);
  h->peer_on = true;
  h->epoch = 0;
  return STCA_OK;
}

extern "C" stca_status stca_ipc_open(const void *ipc_handle, int32_t device, void **ptr_out) {
  if (!ipc_handle || !ptr_out) return STCA_ERR_INVALID_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return STCA_ERR_CUDA;
  cudaIpcMemHandle_t hd;
  memcpy(&hd, ipc_handle, sizeof hd);
  if (cudaIpcOpenMemHandle(ptr_out, hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return STCA_ERR_CUDA;
  }
  return STCA_OK;
}

extern "C" stca_status stca_ipc_close(void *ptr) {
  if (!ptr) return STCA_ERR_INVALID_ARG;
  if (cudaIpcCloseMemHandle(ptr) != cudaSuccess) {
    cudaGetLastError();
    return STCA_ERR_CUDA;
  }
  return STCA_OK;
}

// ===========================================================================
// NEXT-3 (i): the standard attention form, Eq.(12), as a measured variant
// ===========================================================================
extern "C" stca_status stca_set_attention_form(stca_handle *h, int32_t form) {
  if (!h) return STCA_ERR_INVALID_ARG;
  if (form != STCA_FORM_REORDERED && form != STCA_FORM_STANDARD) return fail(h, STCA_ERR_INVALID_ARG, "bad form %d", form);
  if (form == STCA_FORM_REORDERED) {
    h->attn_form = form;
    return STCA_OK;
  }
  const int d = h->cfg.d, hh = h->cfg.h, M = h->cfg.M, dh = d / hh;
  if (!h->bf16 || d != 128)
    return fail(h, STCA_ERR_UNSUPPORTED, "the standard attention form runs on the bf16 path with d = 128 (d=%d)", d);
  CU(cudaSetDevice(h->cfg.device));
  CU(cudaDeviceSynchronize());
  const float c = (float)(1.4426950408889634 / sqrt((double)dh));  // log2(e)/sqrt(d_h): scores in the log2 domain
  std::vector<float> wq((size_t)d * d), wk((size_t)d * d), wv((size_t)d * d), wo((size_t)d * d);
  for (int i = 1; i <= M; ++i) {
    const std::string p = "L" + std::to_string(i) + ".";
    if (!h->std_q[i - 1].WQK) {
      CU(cudaMemcpy(wq.data(), h->w32[p + "WQ"], wq.size() * 4, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(wk.data(), h->w32[p + "WK"], wk.size() * 4, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(wv.data(), h->w32[p + "WV"], wv.size() * 4, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(wo.data(), h->w32[p + "WO"], wo.size() * 4, cudaMemcpyDeviceToHost));
      // per head r a d-column block: Q: [c W_Q^r | 0], KV: [W_K^r | W_V^r | 0]; O: rows of the V block = W_O^r
      std::vector<float> q((size_t)d * hh * d, 0.f), kv((size_t)d * hh * d, 0.f), o((size_t)hh * d * d, 0.f);
      for (int e = 0; e < d; ++e)
        for (int r = 0; r < hh; ++r)
          for (int cc = 0; cc < dh; ++cc) {
            q[(size_t)e * hh * d + r * d + cc] = c * wq[(size_t)e * d + r * dh + cc];
            kv[(size_t)e * hh * d + r * d + cc] = wk[(size_t)e * d + r * dh + cc];
            kv[(size_t)e * hh * d + r * d + dh + cc] = wv[(size_t)e * d + r * dh + cc];
          }
      for (int r = 0; r < hh; ++r)
        for (int cc = 0; cc < dh; ++cc)
          memcpy(&o[((size_t)r * d + dh + cc) * d], &wo[(size_t)(r * dh + cc) * d], sizeof(float) * d);
      void *qd = upload(h, q.data(), q.size()), *kvd = upload(h, kv.data(), kv.size()), *od = upload(h, o.data(), o.size());
      if (!qd || !kvd || !od) return fail(h, STCA_ERR_OOM, "standard-form weight upload failed");
      if (!stca::tc_prepare_layer(qd, od, nullptr, i, d, hh, &h->std_q[i - 1], [&](size_t n) { return dalloc(h, n); }) ||
          !stca::tc_prepare_layer(kvd, nullptr, nullptr, i, d, hh, &h->std_kv[i - 1], [&](size_t n) { return dalloc(h, n); }))
        return fail(h, STCA_ERR_OOM, "standard-form weight repack failed");
    }
  }
  CU(cudaDeviceSynchronize());
  h->attn_form = form;
  return STCA_OK;
}
