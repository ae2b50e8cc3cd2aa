/*
 * stca_oracle.c -- float64 CPU oracle for the STCA forward under RLB.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2511_06077_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or constant with it.
 *
 * What it computes: the plain definition of PAPER.md §3.1 (arXiv 2511.06077),
 *   Eq.(1)  SwiGLUFFN(x) = ((x Wu) ⊙ (x Wv ⊙ sigmoid(x Wv))) Wo
 *   Eq.(2)  X~(i) = LN(SwiGLUFFN(i)(X))
 *   Eq.(3)  q(1)  = LN(SwiGLUFFN(1)(x_t))
 *   Eq.(4)  alpha(i,r) = softmax(q W_Q^r (X~ W_K^r)^T / sqrt(d_h))
 *   Eq.(5)  o(i,r) = alpha (X~ W_V^r)
 *   Eq.(6)  o(i) = [o(i,1) | ... | o(i,h)] W_O
 *   Eq.(7)  q(i+1) = SwiGLUFFN(i+1)([o(1)|...|o(i)|x_t] W_C(i+1))
 *   Eq.(8)  Z_H = [o(1); ...; o(M)]
 *   Eq.(9)  z = SwiGLUFFN_Z([o(1)|...|o(M)|x_t] W_Z)
 * with attention in the STANDARD form (Eq.(12)).  The reordered
 * form (Eq.(13)) is available as form=1 for the dual-form pin.
 *
 * Request-level batching (§3.2): the history path
 * Phi_user(H) -- X~(i) and the per-head K/V projections of the standard form --
 * is computed once per request and reused by all of its targets; every target
 * then runs the identical per-target code, so a request with m targets gives
 * bit-identical results to m single-target requests with the same history.
 *
 * Readings where the paper is silent (DESIGN.md "Readings" R1-R20): no biases
 * (P:L109); LN eps inside the sqrt, biased variance; X~(i) from raw X per
 * layer; max-subtracted softmax; no LN on fused queries; x_t last in the
 * concatenations; head r = columns [r d_h, (r+1) d_h); L_infer keeps the most
 * recent (last) L_infer rows.
 *
 * Arithmetic: float64, scalar loops, ascending-index summation, compiled with
 * -O2 -ffp-contract=off (no FMA contraction).  Threads run over requests only,
 * so results are bit-identical to a serial run.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum {
  ORC_OK = 0, ORC_ERR_INVALID_ARG = -1, ORC_ERR_SHAPE = -2, ORC_ERR_OFFSETS = -3,
  ORC_ERR_EMPTY_HISTORY = -4, ORC_ERR_OOM = -7
};

typedef struct {
  int32_t d, h, r, M;
  int32_t L_infer;  /* >0: keep the last L_infer rows of every history */
  double ln_eps;
  int32_t with_z;
} oracle_cfg;

typedef struct {
  const double *hWu, *hWv, *hWo, *hg, *hb; /* history SwiGLUFFN(i) + LN, Eq.(2) */
  const double *qWu, *qWv, *qWo;          /* query SwiGLUFFN(i): Eq.(3) for i=1, Eq.(7) else */
  const double *qg, *qb;                  /* query LN, Eq.(3) (layer 1 only) */
  const double *WQ, *WK, *WV, *WO;        /* d x d each, head r = cols [r dh,(r+1)dh) */
  const double *WC;                       /* W_C(i): (i d) x d, i >= 2 (NULL for i = 1) */
} oracle_layer;

typedef struct { const double *WZ, *Wu, *Wv, *Wo; } oracle_head;

/* ------------------------------------------------------------------ */
/* primitives                                                          */
/* ------------------------------------------------------------------ */

/* out[n x p] = a[n x k] . w[k x p], ascending-k accumulation per element. */
static void matmul(const double *a, int64_t n, int64_t k, const double *w, int64_t p, double *out) {
  for (int64_t i = 0; i < n; ++i) {
    double *o = out + i * p;
    for (int64_t j = 0; j < p; ++j) o[j] = 0.0;
    for (int64_t kk = 0; kk < k; ++kk) {
      const double av = a[i * k + kk];
      const double *wr = w + kk * p;
      for (int64_t j = 0; j < p; ++j) o[j] += av * wr[j];
    }
  }
}

static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

/* Eq.(1), applied row-wise to x[n x d]; scratch >= 2*r*d doubles. */
void oracle_swigluffn(const double *x, int64_t n, int32_t d, int32_t rd, const double *Wu,
                      const double *Wv, const double *Wo, double *out) {
  double *a = (double *)malloc(sizeof(double) * (size_t)rd * 2);
  double *g = a + rd;
  for (int64_t i = 0; i < n; ++i) {
    matmul(x + i * d, 1, d, Wu, rd, a);          /* x Wu */
    matmul(x + i * d, 1, d, Wv, rd, g);          /* x Wv */
    for (int32_t k = 0; k < rd; ++k) a[k] = a[k] * (g[k] * sigmoid(g[k]));
    matmul(a, 1, rd, Wo, d, out + i * d);        /* (...) Wo */
  }
  free(a);
}

/* LayerNorm over the last axis (reading R3). */
void oracle_layernorm(const double *x, int64_t n, int32_t d, const double *g, const double *b,
                      double eps, double *out) {
  for (int64_t i = 0; i < n; ++i) {
    const double *xr = x + i * d;
    double mu = 0.0, var = 0.0;
    for (int32_t e = 0; e < d; ++e) mu += xr[e];
    mu /= d;
    for (int32_t e = 0; e < d; ++e) var += (xr[e] - mu) * (xr[e] - mu);
    var /= d;
    const double inv = 1.0 / sqrt(var + eps);
    for (int32_t e = 0; e < d; ++e) out[i * d + e] = (xr[e] - mu) * inv * g[e] + b[e];
  }
}

/* max-subtracted softmax (reading R12), ascending-index sum. */
void oracle_softmax(const double *s, int64_t L, double *out) {
  double mx = -INFINITY, l = 0.0;
  for (int64_t j = 0; j < L; ++j) mx = s[j] > mx ? s[j] : mx;
  for (int64_t j = 0; j < L; ++j) { out[j] = exp(s[j] - mx); l += out[j]; }
  for (int64_t j = 0; j < L; ++j) out[j] /= l;
}

/* ------------------------------------------------------------------ */
/* one attention layer, one request (shared history), many queries      */
/* ------------------------------------------------------------------ */

/* Per-request shared history state for one layer (RLB: computed once). */
typedef struct {
  int64_t L;
  const double *Xt;   /* [L x d], X~(i) */
  double *K, *V;      /* standard form: [h][L x dh] = X~ W_K^r, X~ W_V^r */
} hist_state;

static void hist_kv(hist_state *hs, int32_t d, int32_t h, const double *WK, const double *WV,
                    double *colbuf_k, double *colbuf_v) {
  const int32_t dh = d / h;
  /* K_r = X~ W_K[:, C_r]; computed column block by column block. */
  for (int32_t r = 0; r < h; ++r) {
    for (int32_t e = 0; e < d; ++e)
      for (int32_t c = 0; c < dh; ++c) {
        colbuf_k[e * dh + c] = WK[(int64_t)e * d + r * dh + c];
        colbuf_v[e * dh + c] = WV[(int64_t)e * d + r * dh + c];
      }
    matmul(hs->Xt, hs->L, d, colbuf_k, dh, hs->K + (int64_t)r * hs->L * dh);
    matmul(hs->Xt, hs->L, d, colbuf_v, dh, hs->V + (int64_t)r * hs->L * dh);
  }
}

/* Eq.(4)-(6) standard form (form 0) or Eq.(13) reordered form (form 1) for one
 * query q[d] against one request's history; writes o[d]. */
static void attend(const hist_state *hs, const double *q, int32_t d, int32_t h, const double *WQ,
                   const double *WK, const double *WV, const double *WO, int form, double *o,
                   double *s /* [L] */, double *alpha /* [L] */, double *cat /* [d] */,
                   double *tmp /* [2d] */) {
  const int32_t dh = d / h;
  const double scale = 1.0 / sqrt((double)dh);
  const int64_t L = hs->L;
  for (int32_t r = 0; r < h; ++r) {
    double *qh = tmp; /* [dh] = q W_Q[:, C_r] */
    for (int32_t c = 0; c < dh; ++c) qh[c] = 0.0;
    for (int32_t e = 0; e < d; ++e)
      for (int32_t c = 0; c < dh; ++c) qh[c] += q[e] * WQ[(int64_t)e * d + r * dh + c];
    if (form == 0) {
      const double *K = hs->K + (int64_t)r * L * dh, *V = hs->V + (int64_t)r * L * dh;
      for (int64_t j = 0; j < L; ++j) {
        double acc = 0.0;
        for (int32_t c = 0; c < dh; ++c) acc += qh[c] * K[j * dh + c];
        s[j] = acc * scale;
      }
      oracle_softmax(s, L, alpha);
      for (int32_t c = 0; c < dh; ++c) cat[r * dh + c] = 0.0;
      for (int64_t j = 0; j < L; ++j)
        for (int32_t c = 0; c < dh; ++c) cat[r * dh + c] += alpha[j] * V[j * dh + c];
    } else {
      double *u = tmp + dh; /* [d] = (q W_Q^r) W_K^r^T */
      for (int32_t e = 0; e < d; ++e) {
        double acc = 0.0;
        for (int32_t c = 0; c < dh; ++c) acc += qh[c] * WK[(int64_t)e * d + r * dh + c];
        u[e] = acc;
      }
      for (int64_t j = 0; j < L; ++j) {
        double acc = 0.0;
        for (int32_t e = 0; e < d; ++e) acc += u[e] * hs->Xt[j * d + e];
        s[j] = acc * scale;
      }
      oracle_softmax(s, L, alpha);
      double *y = u; /* alpha X~, reuse */
      for (int32_t e = 0; e < d; ++e) y[e] = 0.0;
      for (int64_t j = 0; j < L; ++j)
        for (int32_t e = 0; e < d; ++e) y[e] += alpha[j] * hs->Xt[j * d + e];
      for (int32_t c = 0; c < dh; ++c) {
        double acc = 0.0;
        for (int32_t e = 0; e < d; ++e) acc += y[e] * WV[(int64_t)e * d + r * dh + c];
        cat[r * dh + c] = acc;
      }
    }
  }
  matmul(cat, 1, d, WO, d, o); /* Eq.(6) */
}

/* Single-query, single-layer attention, exported for the pins (P4-P8, P19). */
int oracle_attention(const double *q, const double *Xt, int64_t L, int32_t d, int32_t h,
                     const double *WQ, const double *WK, const double *WV, const double *WO,
                     int form, double *o) {
  if (L <= 0) return ORC_ERR_EMPTY_HISTORY;
  if (d <= 0 || h <= 0 || d % h) return ORC_ERR_SHAPE;
  const int32_t dh = d / h;
  hist_state hs = {L, Xt, NULL, NULL};
  double *buf = (double *)malloc(sizeof(double) * ((size_t)2 * h * L * dh + 2 * L + 3 * (size_t)d + 2 * (size_t)d * dh));
  if (!buf) return ORC_ERR_OOM;
  hs.K = buf;
  hs.V = hs.K + (int64_t)h * L * dh;
  double *s = hs.V + (int64_t)h * L * dh, *alpha = s + L, *cat = alpha + L, *tmp = cat + d,
         *cb = tmp + 2 * d;
  if (form == 0) hist_kv(&hs, d, h, WK, WV, cb, cb + (int64_t)d * dh);
  attend(&hs, q, d, h, WQ, WK, WV, WO, form, o, s, alpha, cat, tmp);
  free(buf);
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* validation + suffix (exact integer work, §8(a) row a0)               */
/* ------------------------------------------------------------------ */

int oracle_validate(const oracle_cfg *cfg, const int64_t *hist_off, const int64_t *tgt_off,
                    int64_t B, int64_t T, int64_t Nt, int64_t *bad_index) {
  *bad_index = -1;
  if (!cfg || B < 0) return ORC_ERR_INVALID_ARG;
  if (cfg->d <= 0 || cfg->h <= 0 || cfg->r < 1 || cfg->M < 1 || cfg->d % cfg->h) return ORC_ERR_SHAPE;
  if (B > 0 && (!hist_off || !tgt_off)) return ORC_ERR_INVALID_ARG;
  if (hist_off[0] != 0 || tgt_off[0] != 0) return ORC_ERR_OFFSETS;
  for (int64_t b = 0; b < B; ++b) {
    if (hist_off[b + 1] < hist_off[b] || tgt_off[b + 1] < tgt_off[b]) { *bad_index = b; return ORC_ERR_OFFSETS; }
  }
  if (hist_off[B] != T || tgt_off[B] != Nt) return ORC_ERR_OFFSETS;
  for (int64_t b = 0; b < B; ++b)
    if (hist_off[b + 1] == hist_off[b]) { *bad_index = b; return ORC_ERR_EMPTY_HISTORY; }
  return ORC_OK;
}

/* Temporal suffix: start'_b = max(off[b], off[b+1] - L_infer). */
void oracle_suffix(const int64_t *hist_off, int64_t B, int32_t L_infer, int64_t *start) {
  for (int64_t b = 0; b < B; ++b) {
    int64_t s = hist_off[b];
    if (L_infer > 0 && hist_off[b + 1] - L_infer > s) s = hist_off[b + 1] - L_infer;
    start[b] = s;
  }
}

/* ------------------------------------------------------------------ */
/* full forward                                                         */
/* ------------------------------------------------------------------ */

typedef struct {
  const oracle_cfg *cfg;
  const oracle_layer *layers;
  const oracle_head *head;
  const double *X, *XT;
  const int64_t *hist_off, *tgt_off, *start;
  int64_t B;
  double *Z, *z;
  int form;
  int64_t next;
  pthread_mutex_t mu;
  int status;
} fwd_job;

static int forward_request(fwd_job *J, int64_t b) {
  const oracle_cfg *cfg = J->cfg;
  const int32_t d = cfg->d, h = cfg->h, M = cfg->M, rd = cfg->r * cfg->d, dh = d / h;
  const int64_t s0 = J->start[b], e0 = J->hist_off[b + 1], L = e0 - s0;
  const int64_t t0 = J->tgt_off[b], t1 = J->tgt_off[b + 1], m = t1 - t0;
  if (m == 0) return ORC_OK;
  size_t need = (size_t)L * d * 2            /* y, Xt */
              + (size_t)2 * h * L * dh       /* K, V */
              + (size_t)2 * L                /* s, alpha */
              + (size_t)m * d                /* q per target */
              + (size_t)m * (M + 1) * d      /* concat [o1..oM | x_t] per target */
              + (size_t)(M + 1) * d          /* c */
              + (size_t)5 * d + (size_t)2 * d * dh;
  double *buf = (double *)malloc(sizeof(double) * need);
  if (!buf) return ORC_ERR_OOM;
  double *y = buf, *Xt = y + L * d, *K = Xt + L * d, *V = K + (int64_t)h * L * dh, *s = V + (int64_t)h * L * dh,
         *alpha = s + L, *q = alpha + L, *catv = q + m * d, *c = catv + m * (M + 1) * d,
         *cat = c + (M + 1) * d, *tmp = cat + d, *o = tmp + 2 * d, *cb = o + d;
  const double *Xb = J->X + s0 * d;

  /* q(1) = LN(SwiGLUFFN(1)(x_t)), Eq.(3) */
  const oracle_layer *L1 = &J->layers[0];
  for (int64_t t = 0; t < m; ++t) {
    oracle_swigluffn(J->XT + (t0 + t) * d, 1, d, rd, L1->qWu, L1->qWv, L1->qWo, c);
    oracle_layernorm(c, 1, d, L1->qg, L1->qb, cfg->ln_eps, q + t * d);
  }
  for (int64_t t = 0; t < m; ++t) /* x_t is the last block of every concatenation (R10) */
    memcpy(catv + t * (M + 1) * d + (int64_t)M * d, J->XT + (t0 + t) * d, sizeof(double) * d);

  for (int32_t i = 1; i <= M; ++i) {
    const oracle_layer *Ly = &J->layers[i - 1];
    /* X~(i) = LN(SwiGLUFFN(i)(X)), Eq.(2), from raw X (R4), once per request (RLB). */
    oracle_swigluffn(Xb, L, d, rd, Ly->hWu, Ly->hWv, Ly->hWo, y);
    oracle_layernorm(y, L, d, Ly->hg, Ly->hb, cfg->ln_eps, Xt);
    hist_state hs = {L, Xt, K, V};
    if (J->form == 0) hist_kv(&hs, d, h, Ly->WK, Ly->WV, cb, cb + (int64_t)d * dh);
    for (int64_t t = 0; t < m; ++t) {
      double *ct = catv + t * (M + 1) * d;
      attend(&hs, q + t * d, d, h, Ly->WQ, Ly->WK, Ly->WV, Ly->WO, J->form, o, s, alpha, cat, tmp);
      memcpy(ct + (int64_t)(i - 1) * d, o, sizeof(double) * d);
      memcpy(J->Z + ((t0 + t) * M + (i - 1)) * d, o, sizeof(double) * d); /* Eq.(8) */
      if (i < M) {
        /* q(i+1) = SwiGLUFFN(i+1)([o(1)..o(i) | x_t] W_C(i+1)), Eq.(7) */
        const oracle_layer *Ln = &J->layers[i];
        double *cin = c; /* [(i+1) d] concatenation, x_t last */
        memcpy(cin, ct, sizeof(double) * (size_t)i * d);
        memcpy(cin + (int64_t)i * d, ct + (int64_t)M * d, sizeof(double) * d);
        double *proj = tmp; /* [d] */
        matmul(cin, 1, (int64_t)(i + 1) * d, Ln->WC, d, proj);
        oracle_swigluffn(proj, 1, d, rd, Ln->qWu, Ln->qWv, Ln->qWo, q + t * d);
      }
    }
  }
  if (cfg->with_z && J->z) {
    /* z = SwiGLUFFN_Z([o(1)..o(M) | x_t] W_Z), Eq.(9) */
    for (int64_t t = 0; t < m; ++t) {
      matmul(catv + t * (M + 1) * d, 1, (int64_t)(M + 1) * d, J->head->WZ, d, tmp);
      oracle_swigluffn(tmp, 1, d, rd, J->head->Wu, J->head->Wv, J->head->Wo, J->z + (t0 + t) * d);
    }
  }
  free(buf);
  return ORC_OK;
}

static void *fwd_worker(void *arg) {
  fwd_job *J = (fwd_job *)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int64_t b = J->next++;
    int st = J->status;
    pthread_mutex_unlock(&J->mu);
    if (b >= J->B || st != ORC_OK) break;
    int rc = forward_request(J, b);
    if (rc != ORC_OK) {
      pthread_mutex_lock(&J->mu);
      J->status = rc;
      pthread_mutex_unlock(&J->mu);
    }
  }
  return NULL;
}

/* Full forward.  layers[M], head (may be NULL if !with_z), X [T x d],
 * XT [Nt x d], Z [Nt x M x d], z [Nt x d] or NULL.  form 0 = standard
 * (definition), 1 = reordered.  Returns ORC_* status; *bad_index names the
 * offending request on OFFSETS / EMPTY_HISTORY. */
int oracle_forward(const oracle_cfg *cfg, const oracle_layer *layers, const oracle_head *head,
                   const double *X, int64_t T, const int64_t *hist_off, int64_t B, const double *XT,
                   int64_t Nt, const int64_t *tgt_off, double *Z, double *z, int form,
                   int32_t nthreads, int64_t *bad_index) {
  int rc = oracle_validate(cfg, hist_off, tgt_off, B, T, Nt, bad_index);
  if (rc != ORC_OK) return rc;
  if (cfg->with_z && z && !head) return ORC_ERR_INVALID_ARG;
  int64_t *start = (int64_t *)malloc(sizeof(int64_t) * (size_t)(B > 0 ? B : 1));
  oracle_suffix(hist_off, B, cfg->L_infer, start);
  fwd_job J;
  J.cfg = cfg; J.layers = layers; J.head = head; J.X = X; J.XT = XT; J.hist_off = hist_off;
  J.tgt_off = tgt_off; J.start = start; J.B = B; J.Z = Z; J.z = z; J.form = form; J.next = 0;
  J.status = ORC_OK;
  pthread_mutex_init(&J.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  for (int i = 1; i < nthreads; ++i) pthread_create(&th[i], NULL, fwd_worker, &J);
  fwd_worker(&J);
  for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
  pthread_mutex_destroy(&J.mu);
  free(start);
  return J.status;
}
