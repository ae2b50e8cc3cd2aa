/*
 * stca.h -- C ABI of the B200-native STCA forward under Request-Level Batching.
 *
 * Method: arXiv 2511.06077, "Make It Long, Keep It Fast".
 *   - Stacked Target-to-History Cross Attention, §3.1 Eq.(1)-(9), P:L95-156,
 *     executed in the reordered single-query form Eq.(13), P:L175-198;
 *   - Request-Level Batching, §3.2: one history per request,
 *     projected once per layer (X~(i), Eq.(2)) and shared by all of that
 *     request's targets;
 *   - ragged histories with an offsets ("index") tensor, capped at the
 *     serving length L_infer by keeping the temporal suffix.
 *
 * Every entry point is extern "C", takes plain pointers and sizes, throws
 * nothing and returns an stca_status.  No torch / C++ types cross it.
 *
 * Threading: a handle is not thread-safe; use one handle per thread / device.
 * Streams are passed as `void*` holding a cudaStream_t (NULL = legacy stream).
 */
#ifndef STCA_H_
#define STCA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STCA_ABI_VERSION 2
#define STCA_MAX_LAYERS 16

typedef enum {
  STCA_OK = 0,
  STCA_ERR_INVALID_ARG = -1,   /* NULL pointer, negative size, bad enum */
  STCA_ERR_SHAPE = -2,         /* d % h != 0, weight shape mismatch (message names both shapes) */
  STCA_ERR_OFFSETS = -3,       /* off[0] != 0, decreasing offsets, or off[B] != rows */
  STCA_ERR_EMPTY_HISTORY = -4, /* L_b == 0: softmax over an empty set (message names b) */
  STCA_ERR_UNSUPPORTED = -5,   /* e.g. bf16 path with d % 16 != 0 */
  STCA_ERR_STATE = -6,         /* forward before project, or B mismatch with the projection */
  STCA_ERR_OOM = -7,           /* device allocation failed */
  STCA_ERR_CUDA = -8,          /* kernel / launch / copy failure (sticky: destroy the handle) */
  STCA_ERR_COMM = -9           /* split-history exchange callback failed */
} stca_status;

typedef enum {
  STCA_BF16 = 0, /* bf16 storage and tensor-core operands, fp32 accumulation and softmax */
  STCA_FP32 = 1  /* fp32 everywhere (CUDA cores, no TF32): the 1e-4 parity path */
} stca_dtype;

/* Split-history exchange: an all-gather of `bytes` bytes
 * from every rank, called once per layer on `stream` with device pointers.
 * recv holds split_world * bytes bytes, rank-major.  Return 0 on success.
 * Optional: handles attached to peer buffers (stca_split_peer_attach) exchange over peer memory
 * instead and never call it. */
typedef int (*stca_exchange_fn)(void *ctx, const void *send, void *recv, size_t bytes, void *stream);

/* Device-memory provider for the handle's WORKING buffers (the projected X~ cache, staging, split-K
 * partials, scratch; weights are allocated once at create with cudaMalloc).  alloc returns `bytes`
 * bytes on `device` usable in stream order on `stream` (NULL on failure -> STCA_ERR_OOM); free
 * releases a pointer from alloc once the work already enqueued on `stream` is done with it (stream
 * order, no device synchronisation).  Buffers only grow, so a steady state of same-sized calls
 * allocates nothing.  Both NULL: the CUDA stream-ordered pool (cudaMallocAsync / cudaFreeAsync).
 * The Python binding passes PyTorch's caching allocator (torch.cuda.caching_allocator_alloc). */
typedef void *(*stca_alloc_fn)(void *ctx, size_t bytes, int32_t device, void *stream);
typedef void (*stca_free_fn)(void *ctx, void *ptr, int32_t device, void *stream);

typedef struct {
  int32_t d, h, r, M;     /* model dim, heads (d % h == 0), SwiGLU ratio r >= 1, layers 1..STCA_MAX_LAYERS */
  int32_t L_infer;        /* > 0: keep the most recent L_infer rows of each history; 0: no cap */
  float ln_eps;           /* LayerNorm eps inside the sqrt (paper silent; 1e-5) */
  int32_t dtype;          /* stca_dtype */
  int32_t with_z;         /* also compute z = SwiGLUFFN_Z([o(1)..o(M)|x_t] W_Z), Eq.(9) */
  int32_t device;         /* CUDA ordinal the handle lives on */
  int32_t chunk_keys;     /* split-K chunk length cap in keys (multiple of 128); 0 = default 8192 */
  int32_t split_rank;     /* split-history mode: this rank, 0..split_world-1 */
  int32_t split_world;    /* 1 = off; > 1: every rank gets the SAME full inputs and owns a */
                          /* contiguous block of key chunks of every history */
  stca_exchange_fn exchange; /* split-history without peer buffers: the per-layer all-gather */
  void *exchange_ctx;
  stca_alloc_fn dev_alloc; /* NULL: stream-ordered CUDA pool (see stca_alloc_fn) */
  stca_free_fn dev_free;
  void *alloc_ctx;
} stca_config;

/* A named weight, HOST memory, float32, row-major in the paper's row-vector
 * orientation [in x out] (y = x W).  Values are rounded to bf16 (RNE) on the
 * bf16 path.  Names (i = 1..M):
 *   L{i}.hist.{Wu,Wv}  d x rd   L{i}.hist.Wo  rd x d   L{i}.hist.{ln_g,ln_b} 1 x d   Eq.(1)-(2)
 *   L{i}.qry.{Wu,Wv,Wo}        (query SwiGLUFFN(i): Eq.(3) for i = 1, Eq.(7) for i >= 2)
 *   L1.qry.{ln_g,ln_b}         (LN of Eq.(3))
 *   L{i}.{WQ,WK,WV,WO} d x d   head r = columns [r d/h, (r+1) d/h); WO rows in head order
 *   L{i}.WC (i d) x d, i >= 2  (W_C(i) of Eq.(7); concatenation [o(1)|..|o(i-1)|x_t])
 *   z.WZ ((M+1) d) x d, z.{Wu,Wv,Wo}   (only with with_z)
 * Reading R5 (shared FFN): pass the same data pointer for hist and qry. */
typedef struct {
  const char *name;
  const float *data;
  int64_t rows, cols;
} stca_tensor;

typedef struct stca_handle stca_handle;

/* Validates cfg and every weight (missing / duplicate / mis-shaped names ->
 * SHAPE or INVALID_ARG with the names and both shapes in the message), copies
 * and repacks them into handle-owned device memory on cfg->device.  The
 * caller may free its buffers on return.  Precomputes, per layer and head,
 * W_QK^r = W_Q^r W_K^r^T (the reordered query map) and
 * W_VO^r = W_V^r W_O^r (so o = sum_r (alpha_r X~) W_VO^r, Eq.(13) + Eq.(6)). */
stca_status stca_create(const stca_config *cfg, const stca_tensor *weights, int32_t n_weights,
                        stca_handle **out);

/* History path, Eq.(2), once per request (RLB):
 *   X~(i) = LN(SwiGLUFFN(i)(X_b[start'_b:end_b]))  for every layer i and request b,
 * start'_b = max(hist_off[b], hist_off[b+1] - L_infer).  X is [T x d] row-major,
 * bf16 (uint16 bit patterns) or fp32 per cfg.dtype, rows chronological (oldest
 * first), device OR host memory.  A host X (pinned for asynchrony) is streamed
 * up in pieces on a handle-owned copy stream that waits only for the previous
 * call's reads of the staging buffer, and each piece is projected on `stream`
 * as soon as it has landed (the upload overlaps the projection and any earlier
 * work on `stream`); with L_infer truncation it is staged whole on `stream`.
 * A host X must stay valid and unmodified until `stream` has completed this
 * call's work.  hist_off is a HOST int64 array [B+1], consumed before return.
 * The call does not wait for the device: host-side plans travel through a ring
 * of pinned staging slots, each reused only after the event of its previous
 * copy (so at most 8 calls may be in flight before the host waits).
 * The handle owns the projected cache until the next call or destroy.  On a
 * validation error nothing is enqueued; on any later failure the handle has no
 * projection (stca_forward returns STATE until the next successful call). */
stca_status stca_project_history(stca_handle *h, const void *X, int64_t T, const int64_t *hist_off,
                                 int64_t B, void *stream);

/* Target path for the B requests of the last projection, Eq.(3)-(9):
 * xt [Nt x d] (dtype per cfg, device or host), tgt_off HOST int64 [B+1]
 * (request b owns target rows [tgt_off[b], tgt_off[b+1]); m_b = 0 is legal).
 * Outputs (device or host, float32): out_Z [Nt x M x d] = Z_H rows (Eq.(8)),
 * out_z [Nt x d] or NULL.  Everything is enqueued on `stream` and the call does
 * not wait for the device (the work list reaches it through the pinned staging
 * ring above): host inputs must stay valid and host outputs are complete only
 * once `stream` has completed this call's work (use pinned memory for
 * asynchrony).  Any number of forwards may reuse one projection. */
stca_status stca_forward(stca_handle *h, const void *xt, int64_t Nt, const int64_t *tgt_off, int64_t B,
                         float *out_Z, float *out_z, void *stream);

/* ---- session sharing: RLB extended across requests of the same user ----
 * PAPER.md P:L45 ("can be extended to share across multiple requests for the same user/session") and
 * P:L51 ("multi-request sharing for the same user/session").  stca_session_open gives the handle a
 * persistent X~ cache of `capacity_rows` history rows per layer (M x capacity x d, storage dtype) and
 * forgets any earlier projection.  stca_project_history_session then does what stca_project_history
 * does for B requests of users user_id[b] (HOST int64 [B]) whose history has generation gen[b] (HOST
 * int64 [B]; any caller value that changes whenever the user's kept rows change, e.g. the newest
 * event's timestamp) -- except that a request whose (user, generation, kept length L'_b) is cached is
 * not projected again: the following stca_forward calls attend over the cached rows, which are the
 * same bits a fresh projection writes (the projection is row-wise).  The missing users' suffix rows
 * are projected into one contiguous range of a FIFO ring; entries it overlaps are forgotten (if that
 * would drop a hit of this batch, the cache is reset and the batch projected whole).  X, T and
 * hist_off as in stca_project_history (every request's rows are passed; rows of hits are not read).
 * *n_projected (may be NULL) = users projected by this call.  STATE before stca_session_open;
 * INVALID_ARG for a user twice in one batch with different histories; OOM when the batch's new rows
 * exceed the capacity; UNSUPPORTED in split-history mode.  A plain stca_project_history closes the
 * session. */
stca_status stca_session_open(stca_handle *h, int64_t capacity_rows, void *stream);
stca_status stca_project_history_session(stca_handle *h, const int64_t *user_id, const int64_t *gen, const void *X,
                                         int64_t T, const int64_t *hist_off, int64_t B, int64_t *n_projected,
                                         void *stream);

/* The projected history cache of the last stca_project_history, Eq.(2): rows [row0, row0 + nrows)
 * of X~(layer), layer = 1..M, in compacted cache order (request b's kept rows start at the sum of
 * the kept lengths L'_{b'} of the requests before it), widened to float32 into out [nrows x d]
 * (device or host; a host copy completes before return).  STATE before any projection,
 * INVALID_ARG for a layer or row range outside the cache. */
stca_status stca_read_cache(stca_handle *h, int32_t layer, int64_t row0, int64_t nrows, float *out, void *stream);

/* ---- per-phase device timing (bench.py's roofline evidence) ----
 * enable != 0: every later project / forward call records CUDA events on its stream around each
 * phase: STCA_PH_PROJECT (a1, the history projection), STCA_PH_ATTENTION (a4: the attention
 * launches of one layer = one region), STCA_PH_MERGE (the split-K fold of one layer),
 * STCA_PH_TARGET (a2/a3/a5-a7: the target-side GEMM launches, one region per launch) and
 * STCA_PH_FORWARD (a whole stca_forward).  Events between kernels remove the programmatic-
 * dependent-launch overlap across them, so profiled phase times are upper bounds of unprofiled
 * ones.  stca_profile_read waits for the recorded events, writes the total milliseconds and the
 * region count of every phase since the last read (arrays of STCA_PH_N) and resets.
 * `enable` is a bit mask: STCA_PROF_EVENTS (the project / attention / merge / forward regions),
 * STCA_PROF_EVENTS_TARGET (also a region around every target-side GEMM launch: more perturbation),
 * STCA_PROF_TWICE_ATTENTION / STCA_PROF_TWICE_PROJECT (every a4 / a1 launch is issued twice with
 * identical results -- a diagnostic: the step-time difference is the launches' marginal cost, which
 * power management inflates, so the bench does not use it as a kernel duration). */
enum { STCA_PH_PROJECT = 0, STCA_PH_ATTENTION = 1, STCA_PH_MERGE = 2, STCA_PH_TARGET = 3, STCA_PH_FORWARD = 4,
       STCA_PH_N = 5 };
enum { STCA_PROF_EVENTS = 1, STCA_PROF_TWICE_ATTENTION = 2, STCA_PROF_TWICE_PROJECT = 4, STCA_PROF_EVENTS_TARGET = 8 };
stca_status stca_profile(stca_handle *h, int32_t enable);
stca_status stca_profile_read(stca_handle *h, double *ms, int64_t *count);

void stca_destroy(stca_handle *h);                  /* NULL-safe; synchronises the device */
const char *stca_last_error(const stca_handle *h);  /* last non-OK message; h == NULL: last failed create on this thread */
const char *stca_status_string(int32_t status);
int32_t stca_abi_version(void);
int64_t stca_kernel_launches(void);                  /* process-wide count of kernels libstca has launched */

/* ---- host planning, exposed for exact (bit-for-bit) tests; no device needed ---- */

/* Same validation as project/forward (0 or a negative status); *bad_index = b for
 * OFFSETS/EMPTY_HISTORY, else -1. */
stca_status stca_validate_offsets(const int64_t *hist_off, const int64_t *tgt_off, int64_t B, int64_t T,
                                  int64_t Nt, int64_t *bad_index);

/* start'_b for b < B. */
void stca_plan_suffix(const int64_t *hist_off, int64_t B, int32_t L_infer, int64_t *start_out);

/* Split-K chunk plan of one history of L keys: returns the chunk count and
 * writes the chunk length (a function of L and chunk_keys only). */
int32_t stca_plan_chunks(int64_t L, int32_t chunk_keys, int64_t *chunk_len);

/* Attention work list (request, first query row, query rows, first key, key count,
 * chunk index) as 6 int64 per item in launch order; returns the item count, or the
 * required count if it exceeds `cap`.  m_b h query rows per request, tiles of
 * `qtile` rows. */
int64_t stca_plan_attention(const int64_t *hist_len, const int64_t *tgt_off, int64_t B, int32_t h,
                            int32_t qtile, int32_t chunk_keys, int64_t *items, int64_t cap);

/* Split-history ownership: rank g of G owns the contiguous key range [*own0, *own0 + *olen) of a
 * history of L keys -- the chunks c with floor(c G / C) == g of its stca_plan_chunks plan. */
void stca_plan_split(int64_t L, int32_t chunk_keys, int32_t G, int32_t g, int64_t *own0, int64_t *olen);

/* LPT partition of requests over n_parts GPUs by cost (descending cost to the
 * least-loaded part, ties to the lowest index; exact integer arithmetic).
 * part_out[b] in [0, n_parts). */
void stca_plan_shards(const int64_t *cost, int64_t B, int32_t n_parts, int32_t *part_out);

/* Persistent-kernel schedule: n work items of `cost` over n_ctas CTAs by the LPT rule of
 * stca_plan_shards (bin_out[i] = CTA of item i), written as CSR into cta_list:
 * [n_ctas + 1] offsets, then the item indices of each CTA in descending cost (ties by index). */
void stca_plan_persistent(const int64_t *cost, int64_t n, int32_t n_ctas, int32_t *cta_list, int32_t *bin_out);

/* ---- training data path into the ragged forward ----
 * PAPER.md §3.3 "Subsequence selection" / "Batch-Level Load Balancing"; the
 * algorithmic readings are DESIGN.md R-N2a (rounding) and R-N2b (allocation rule).  All pointers
 * are DEVICE pointers owned by the caller; work is ordered on `stream` (NULL: legacy stream). */

/* Per request b < B: L_train_b = 8 * floor((L_min + s_b (L_max - L_min)) / 8 + 1/2) (Eq. beta-scale
 * P:L258 + P:L260, fp64; s_b ~ Beta(alpha, beta) drawn by the caller, in [0, 1]); the temporal suffix
 * request req_b = min(L_train_b, n_b), n_b = hist_off[b+1] - hist_off[b]; the global length
 * allocation alloc[b] <= req_b with sum(alloc) <= B * L_avg; new_off [B+1] = exclusive
 * prefix sum of alloc, the ragged index over the compacted rows.
 * Synchronises `stream` (reads a device status word).  INVALID_ARG for B outside [1, 49152],
 * L_min > L_max, L_avg < 1, an s_b outside [0, 1] or an infeasible budget (sum of min(req_b, 8) >
 * B * L_avg); alloc/new_off are then unspecified.  CUDA on a launch failure. */
stca_status stca_rlb_allocate(const double *s, const int64_t *hist_off, int64_t B, int32_t L_min, int32_t L_max,
                              int32_t L_avg, int64_t *alloc, int64_t *new_off, void *stream);

/* Sequence compaction: the last alloc[b] rows of request b's history in X [T x row_bytes]
 * (rows hist_off[b+1] - alloc[b] .. hist_off[b+1] - 1) are copied, back to back in request order, to
 * P [new_off[B] x row_bytes], viewed as physical rows of L_avg tokens laid end to end.  The segment
 * map: segs [n_seg x 3] int64 (row, start, len) triples, those of request b at seg_off[b] ..
 * seg_off[b+1] - 1 (seg_off [B+1]); n_seg <= 2B when new_off[B] <= B * L_avg (capacity the caller
 * provides).  alloc/new_off as written by stca_rlb_allocate.  row_bytes a positive multiple of 16, X
 * and P 16-byte aligned, else INVALID_ARG.  Asynchronous (no host sync); rows are copied bit for bit. */
stca_status stca_rlb_compact(const void *X, int64_t row_bytes, const int64_t *hist_off, const int64_t *alloc,
                             const int64_t *new_off, int64_t B, int32_t L_avg, void *P, int64_t *seg_off,
                             int64_t *segs, void *stream);

/* ---- backward of one layer's attention (partial) ----
 * PAPER.md Eq.(14) trains the stack end to end; RLB aggregates the gradients of a
 * request's shared history before they leave the request.  For layer `layer` of the
 * last projection (bf16 path, d = 128): given the forward's reordered queries U (DEVICE bf16 [N_t h x d],
 * row t h + r, pre-scaled by log2(e)/sqrt(d_h); e.g. from the forward) and dY = dLoss/dY (DEVICE fp32
 * [N_t h x d]), writes
 *   dXt (DEVICE fp32 [T' x d], the X~ cache's compacted row order: request b's kept rows from its
 *        offset, see stca_read_cache): dX~_b = alpha^T dY_b + dS^T U_b -- summed over ALL of the
 *        request's target-head rows inside the kernel (rows of requests without targets: 0),
 *   dU (DEVICE fp32 [N_t h x d]): dS X~_b,
 * with alpha = softmax(ln 2 * U_b X~_b^T), D = rowsum(alpha (dY X~_b^T)), dS = ln 2 alpha (dY X~_b^T - D).
 * A request with more than 64 target-head rows adds its blocks' dX~ with fp32 atomics (the last bits
 * then depend on their order).  Asynchronous on `stream`.  STATE without a projection or for a B
 * mismatch, UNSUPPORTED off the bf16 d = 128 path or in split-history mode, INVALID_ARG otherwise. */
stca_status stca_attention_backward(stca_handle *h, int32_t layer, const void *U, const float *dY,
                                    const int64_t *tgt_off, int64_t B, float *dXt, float *dU, void *stream);

/* Backward of layer `layer`'s history path, Eq.(1)-(2): X~ = LN(SwiGLUFFN(X)) over the
 * rows the last projection kept (bf16 path).  X: DEVICE bf16 [rows x d], those rows in cache order
 * (X itself when nothing was truncated; rows must equal the cache's row count).  Given dXt = dLoss/dX~
 * (DEVICE fp32 [rows x d], e.g. from stca_attention_backward), ACCUMULATES dX += dLoss/dX (DEVICE fp32
 * [rows x d]; sum over the layers by calling once per layer) and WRITES the layer's weight gradients
 * dWu, dWv [d x rd], dWo [rd x d], dgamma, dbeta [d] (DEVICE fp32, the weights' [in x out] orientation).
 * The forward is recomputed (no activations are kept) on the library's tcgen05 GEMMs (the SwiGLU in the
 * epilogue), the SwiGLU-gate backward runs in the epilogue of a tcgen05 GEMM that recomputes X [Wu | Wv],
 * the LayerNorm backward on a kernel of the library, dH / dX / the weight gradients on cuBLAS (bf16
 * operands, fp32 accumulation).  Each history row appears once
 * per request however many targets share it: the gradients are aggregated at the request level.
 * Asynchronous on `stream`.  STATE without a projection, SHAPE for a row-count mismatch, UNSUPPORTED off
 * the bf16 path or over a session cache. */
stca_status stca_history_backward(stca_handle *h, int32_t layer, const void *X, int64_t rows, const float *dXt,
                                  float *dX, float *dWu, float *dWv, float *dWo, float *dgamma, float *dbeta,
                                  void *stream);

/* ---- backward of the WHOLE stack ----
 * PAPER.md Eq.(14) trains the stack of Eq.(2)-(9) end to end; under RLB the gradients of a
 * request's shared history are aggregated over its targets inside the request.  For the
 * last projection (bf16 path, d = 128, no split-history, no session cache): runs the forward over x_t
 * (DEVICE bf16 [N_t x d], as stca_forward; Z_H into out_Z, DEVICE fp32 [N_t x M x d], or internal scratch
 * when NULL) keeping every layer's U and Y, then the vector-Jacobian product of
 *     loss = sum(dZ * Z_H) + sum(dz * z)      (dZ DEVICE fp32 [N_t x M x d]; dz DEVICE fp32 [N_t x d] or NULL)
 * and WRITES
 *   - for every stca_grad {name, grad} given: d loss / d weight role `name` (the names and [rows x cols]
 *     of stca_create's weights; DEVICE fp32, same orientation).  Gradients are per ROLE: where one
 *     parameter serves several roles (the shared-FFN reading passes a layer's history FFN as its query
 *     FFN), its gradient is the sum of its roles'.  Roles not listed are computed into scratch.
 *   - dX (DEVICE fp32 [rows x d] or NULL): d loss / d X over the rows the projection kept, in cache order
 *     (X: DEVICE bf16, those rows, as stca_history_backward; rows must equal the cache's row count);
 *   - dxt (DEVICE fp32 [N_t x d] or NULL): d loss / d x_t.
 * Per layer, from the last: target-side GEMMs of Eq.(6)-(7) (cuBLAS, fp32 storage, TF32 tensor cores), the attention backward
 * (tcgen05 kernel, dX~ summed over the request's target-head rows inside the MMA), the history path's
 * LN + SwiGLU-FFN backward (stca_history_backward's kernels).  Asynchronous on `stream`.  STATE without a
 * projection or for a B mismatch; UNSUPPORTED off the bf16 d = 128 path, in split-history mode or over a
 * session cache; SHAPE for a row-count mismatch; INVALID_ARG for an unknown / duplicate gradient name,
 * NULL or host buffers.  Nothing is enqueued on an error found before the first launch. */
typedef struct {
  const char *name; /* a weight role of stca_create, e.g. "L2.WC", "L1.hist.ln_g", "z.Wo" */
  float *grad;      /* DEVICE fp32, rows x cols of that role */
} stca_grad;
stca_status stca_backward(stca_handle *h, const void *xt, int64_t Nt, const int64_t *tgt_off, int64_t B,
                          const void *X, int64_t rows, const float *dZ, const float *dz, const stca_grad *grads,
                          int32_t n_grads, float *dX, float *dxt, float *out_Z, void *stream);

/* ---- input-encoding prologue ----
 * PAPER.md §3.1.1 "Input encoding" (video, action-type and position embeddings fused into x_j)
 * and the time-delta side information (request time minus item timestamp); additive fusion as
 * in SPEC S:L130-138.  Every pointer below is DEVICE memory owned by the caller (the struct itself is
 * host memory), tables row-major in the storage dtype (bf16 bit patterns or fp32), 16-byte aligned:
 *   video    [n_video + 1 x d]   row n_video: every id outside [0, n_video) (out of vocabulary)
 *   action   [n_action + 1 x d]  row n_action: out of vocabulary
 *   position [n_position x d]    recency rank p_j = (last row of the request) - j, clamped to n_position - 1
 *   tdelta   [n_tdelta x d] or NULL: bucket floor(log2(req_time[b] - timestamp[j])) for a delta >= 1 s,
 *                                    0 otherwise, clamped to n_tdelta - 1
 * (readings R-N4a-c; the paper fixes none of the three). */
typedef struct {
  const void *video;
  int64_t n_video;
  const void *action;
  int64_t n_action;
  const void *position;
  int64_t n_position;
  const void *tdelta;
  int64_t n_tdelta;
} stca_embed_tables;

/* X [T x d] (storage dtype) for the ragged batch hist_off [B+1] (device int64): x_j = video[v'_j] +
 * action[a'_j] + position[p_j] (+ tdelta[bucket_j]) summed in fp32 in that order, rounded once.
 * video_id / action_id / timestamp int64 [T], req_time int64 [B] (timestamp / req_time may be NULL
 * without a tdelta table).  The result feeds stca_project_history directly.  Asynchronous on
 * `stream`.  INVALID_ARG for NULL / negative / misaligned arguments, UNSUPPORTED if d * element size
 * is not a multiple of 16 bytes. */
stca_status stca_encode_history(const stca_embed_tables *tables, int32_t d, int32_t dtype, const int64_t *video_id,
                                const int64_t *action_id, const int64_t *timestamp, const int64_t *hist_off,
                                const int64_t *req_time, int64_t B, int64_t T, void *X, void *stream);

/* ---- split-history over peer memory (the LSE merge of P:L289's key chunks over
 * NVLink / NVSwitch without a collective library) ----
 * Every rank of a split-history group (split_world = G >= 2) exports ONE exchange buffer of
 * 4096 + 2 * capacity_bytes bytes (cudaMalloc on the handle's device; capacity rounded up to 4 KB):
 * 4 KB of epoch flags, then two slots for the per-layer partials (the layer's (O/l, m, l) rows of the
 * chunks it owns, alternating by layer).  After every rank has exported, each one attaches the G
 * buffers in rank order (its own at bases[split_rank]; a peer's buffer mapped into this process, e.g.
 * by stca_ipc_open of the handle the peer exported).  From then on every stca_forward runs, per layer:
 * attention into this layer's slot -> a one-thread kernel publishes the layer's epoch to every peer
 * (a system-scope release store into the peer's flag word) and waits until every peer has published it
 * -> the merge folds each chunk reading it IN PLACE from its owner's slot over NVLink (L2-only loads).  A slot
 * is rewritten two layers later, which every peer's merge of the layer in between proves safe, so no
 * second flag exists.  All waits run on the device (one spinning thread per rank; a watchdog traps
 * after 30 s without a peer, which surfaces as STCA_ERR_CUDA): the host never blocks and the step stays
 * graph-capturable.
 * Every rank must issue the same sequence of stca_forward calls; all ranks must stop using the buffers
 * (e.g. a barrier) before any of them calls stca_destroy.
 *
 * stca_split_peer_export: *base_out = the buffer (DEVICE); ipc_handle_out (64 bytes, a
 *   cudaIpcMemHandle_t) or NULL.  STATE if not in split-history mode or already exported; OOM.
 * stca_split_peer_attach: bases = G DEVICE pointers valid in this process.  INVALID_ARG if
 *   bases[split_rank] is not the exported buffer; STATE before export.  A forward whose partials exceed
 *   capacity_bytes fails with INVALID_ARG before any launch.
 * stca_ipc_open / stca_ipc_close: map / unmap a peer's exported buffer (cudaIpcOpenMemHandle with lazy
 *   peer access) on `device`.  STCA_ERR_CUDA on failure. */
stca_status stca_split_peer_export(stca_handle *h, int64_t capacity_bytes, void **base_out, void *ipc_handle_out);
stca_status stca_split_peer_attach(stca_handle *h, void *const *bases);
stca_status stca_ipc_open(const void *ipc_handle, int32_t device, void **ptr_out);
stca_status stca_ipc_close(void *ptr);

/* ---- NEXT-3 (i): the STANDARD attention form as a variant (Eq.(12),
 * P:L177-182, against the reordered Eq.(13)) ----
 * STCA_FORM_REORDERED (default): u = q W_Q^r W_K^r^T, attention over X~ itself, o = sum_r (alpha_r X~) W_V^r W_O^r.
 * STCA_FORM_STANDARD: per layer the history's K^r = X~ W_K^r and V^r = X~ W_V^r are materialised for
 * every head ([K^r | V^r | 0] in a d-column block per head, one tcgen05 GEMM, T' x h d bf16 in HBM), the
 * query is q W_Q^r, the attention runs per (request, head) on the transposed tcgen05 kernel, and
 * o = sum_r (alpha_r V^r) W_O^r.  Same function (P8 of the oracle pins), different cost: the form the
 * paper's reordering argument is measured against.  bf16 path, d = 128, at most 64 targets per request,
 * no split-history; UNSUPPORTED otherwise (checked here or at the forward).  Takes effect for the next
 * stca_forward; the first switch to STANDARD builds its weights (synchronous). */
#define STCA_FORM_REORDERED 0
#define STCA_FORM_STANDARD 1
stca_status stca_set_attention_form(stca_handle *h, int32_t form);

#ifdef __cplusplus
}
#endif
#endif /* STCA_H_ */
