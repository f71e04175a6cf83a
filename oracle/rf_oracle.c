/* TEST INFRASTRUCTURE ONLY — CPU oracle; see rf_oracle.h for the contract and
 * the reference lines each function restates. Never linked into librf_cuda. */
#define _GNU_SOURCE
#include "rf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ rounding --- */

float rfo_round_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return x; /* NaN */
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

float rfo_round_e4m3(float xf) {
  double x = (double)xf;
  if (isnan(x)) return xf;
  double ax = fabs(x);
  if (isinf(ax)) ax = 448.0; /* satfinite */
  double q;
  if (ax >= 0.015625) { /* normal range: 2^-6 */
    int e;
    frexp(ax, &e); /* ax = f * 2^e, f in [0.5,1) -> unbiased exponent e-1 */
    q = ldexp(1.0, (e - 1) - 3);
  } else {
    q = ldexp(1.0, -9); /* subnormal quantum */
  }
  double r = nearbyint(ax / q) * q; /* exact scaling; RNE under default mode */
  if (r > 448.0) r = 448.0;
  return (float)(x < 0 ? -r : r);
}

void rfo_round_bf16_array(const double* in, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = (double)rfo_round_bf16((float)in[i]);
}

void rfo_round_e4m3_array(const double* in, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = (double)rfo_round_e4m3((float)in[i]);
}

/* ---------------------------------------------------------- row threads --- */

typedef void (*row_fn)(void* ctx, int64_t r);
typedef struct {
  row_fn fn;
  void* ctx;
  int64_t rows;
  int64_t next;
  pthread_mutex_t mu;
} row_pool;

static void* row_worker(void* arg) {
  row_pool* p = (row_pool*)arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    int64_t r = p->next++;
    pthread_mutex_unlock(&p->mu);
    if (r >= p->rows) break;
    p->fn(p->ctx, r);
  }
  return NULL;
}

static void for_rows(row_fn fn, void* ctx, int64_t rows, int threads) {
  if (threads <= 1 || rows < 2) {
    for (int64_t r = 0; r < rows; ++r) fn(ctx, r);
    return;
  }
  if (threads > 256) threads = 256;
  row_pool p = {fn, ctx, rows, 0, PTHREAD_MUTEX_INITIALIZER};
  pthread_t tid[256];
  for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, row_worker, &p);
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* ------------------------------------------------------- safe softmax --- */

void rfo_safe_softmax(const double* x, int64_t rows, int64_t n, double* d1, double* d2) {
  for (int64_t r = 0; r < rows; ++r) {
    const double* xr = x + r * n;
    double m = xr[0];
    for (int64_t i = 0; i < n; ++i) m = fmax(m, xr[i]); /* workloads.cpp:53-55 */
    double t = 0;
    for (int64_t i = 0; i < n; ++i) t += exp(xr[i] - m); /* :56-57 */
    d1[r] = m;
    d2[r] = t;
  }
}

/* ---------------------------------------------------------- attention --- */

typedef struct {
  const double *q, *k, *v;
  int64_t sq, skv, hd;
  double scale;
  double *m, *l, *o;
} attn_ctx;

static void attn_row(void* vctx, int64_t row) {
  attn_ctx* c = (attn_ctx*)vctx;
  int64_t b = row / c->sq;
  const double* qr = c->q + row * c->hd;
  const double* kb = c->k + b * c->skv * c->hd;
  const double* vb = c->v + b * c->skv * c->hd;
  double* p = (double*)malloc(sizeof(double) * (size_t)c->skv);
  /* P = q . K^T (workloads.cpp:86-93), scaled */
  for (int64_t l = 0; l < c->skv; ++l) {
    double acc = 0;
    for (int64_t d = 0; d < c->hd; ++d) acc += qr[d] * kb[l * c->hd + d];
    p[l] = acc * c->scale;
  }
  /* oracle form (workloads.cpp:101-118) */
  double m = p[0];
  for (int64_t l = 0; l < c->skv; ++l) m = fmax(m, p[l]);
  double t = 0;
  for (int64_t l = 0; l < c->skv; ++l) t += exp(p[l] - m);
  double* o = c->o + row * c->hd;
  for (int64_t f = 0; f < c->hd; ++f) o[f] = 0.0;
  for (int64_t l = 0; l < c->skv; ++l) {
    double w = exp(p[l] - m) / t;
    for (int64_t f = 0; f < c->hd; ++f) o[f] += w * vb[l * c->hd + f];
  }
  c->m[row] = m;
  c->l[row] = t;
  free(p);
}

void rfo_attention(const double* q, const double* k, const double* v, int64_t bh,
                   int64_t sq, int64_t skv, int64_t hd, double softmax_scale,
                   double* m, double* l, double* o, int threads) {
  attn_ctx c = {q, k, v, sq, skv, hd, softmax_scale, m, l, o};
  for_rows(attn_row, &c, bh * sq, threads);
}

/* One streamed partial state of the attention cascade. */
typedef struct {
  double m, t;
  int touched;
} attn_state;

/* incr_ingest_element for the attention cascade (simulator.cpp:566-589):
 * snap = (m,t); r1 max folds; r2 corrected by exp(d1'-d1) then += exp(P-d1);
 * r3 corrected by exp(d1'-d1)*d2'/d2 then += exp(P-d1)/d2*V. Corrections are
 * skipped on untouched lanes (apply_factor, simulator.cpp:324-339). */
static void attn_ingest(attn_state* s, double* o, double p, const double* v, int64_t hd) {
  double m_prev = s->m, t_prev = s->t;
  int was = s->touched;
  double m = fmax(m_prev, p);
  double t = was ? t_prev * exp(m_prev - m) : t_prev;
  t += exp(p - m);
  double corr = was ? exp(m_prev - m) * t_prev / t : 1.0;
  double w = exp(p - m) / t;
  for (int64_t f = 0; f < hd; ++f) o[f] = (was ? o[f] * corr : o[f]) + w * v[f];
  s->m = m;
  s->t = t;
  s->touched = 1;
}

/* incr_push_child for the attention cascade (simulator.cpp:592-608). */
static void attn_push(attn_state* r, double* ro, const attn_state* c, const double* co,
                      int64_t hd) {
  if (!c->touched) return;
  double m_prev = r->m, t_prev = r->t;
  int was = r->touched;
  double m = fmax(m_prev, c->m);
  double t = was ? t_prev * exp(m_prev - m) : t_prev;
  t += c->t * exp(c->m - m);
  double corr_r = was ? exp(m_prev - m) * t_prev / t : 1.0;
  double corr_c = exp(c->m - m) * c->t / t;
  for (int64_t f = 0; f < hd; ++f) ro[f] = (was ? ro[f] * corr_r : ro[f]) + co[f] * corr_c;
  r->m = m;
  r->t = t;
  r->touched = 1;
}

int rfo_attention_incremental(const double* p, const double* v, int64_t rows, int64_t kv,
                              int64_t hd, int64_t segments, double* m, double* l,
                              double* o) {
  if (segments < 1 || kv % segments != 0) return -2; /* simulator.cpp:668-671 */
  int64_t slice = kv / segments;
  double* po = (double*)malloc(sizeof(double) * (size_t)hd);
  for (int64_t r = 0; r < rows; ++r) {
    const double* pr = p + r * kv;
    const double* vr = v + r * kv * hd;
    attn_state root = {-INFINITY, 0.0, 0};
    double* ro = o + r * hd;
    for (int64_t f = 0; f < hd; ++f) ro[f] = 0.0;
    for (int64_t s = 0; s < segments; ++s) {
      attn_state part = {-INFINITY, 0.0, 0};
      for (int64_t f = 0; f < hd; ++f) po[f] = 0.0;
      for (int64_t i = s * slice; i < (s + 1) * slice; ++i)
        attn_ingest(&part, po, pr[i], vr + i * hd, hd);
      if (segments == 1) { /* run_incremental: the level-1 state is the root */
        root = part;
        memcpy(ro, po, sizeof(double) * (size_t)hd);
      } else {
        attn_push(&root, ro, &part, po, hd);
      }
    }
    m[r] = root.m;
    l[r] = root.t;
  }
  free(po);
  return 0;
}

void rfo_attention_merge(const double* part_m, const double* part_l, const double* part_o,
                         int64_t nslices, int64_t rows, int64_t hd, double* m, double* l,
                         double* o) {
  for (int64_t r = 0; r < rows; ++r) {
    attn_state root = {-INFINITY, 0.0, 0};
    double* ro = o + r * hd;
    for (int64_t f = 0; f < hd; ++f) ro[f] = 0.0;
    for (int64_t s = 0; s < nslices; ++s) {
      attn_state c = {part_m[s * rows + r], part_l[s * rows + r], 1};
      if (c.t == 0.0 && isinf(c.m) && c.m < 0) c.touched = 0; /* empty slice */
      attn_push(&root, ro, &c, part_o + (s * rows + r) * hd, hd);
    }
    m[r] = root.m;
    l[r] = root.t;
  }
}

/* ------------------------------------------------------------- quant --- */

typedef struct {
  const double *a, *w;
  int64_t K, N, tile_k;
  double fmax;
  double *d1, *c;
} quant_ctx;

static void quant_row(void* vctx, int64_t row) {
  quant_ctx* q = (quant_ctx*)vctx;
  const double* ar = q->a + row * q->K;
  double amax = 0; /* workloads.cpp:194-195 */
  for (int64_t l = 0; l < q->K; ++l) amax = fmax(amax, fabs(ar[l]));
  double* cr = q->c + row * q->N;
  for (int64_t f = 0; f < q->N; ++f) cr[f] = 0.0;
  for (int64_t l = 0; l < q->K; ++l) { /* :198-205 */
    double qv = q->fmax * ar[l] / amax;
    const double* wr = q->w + l * q->N;
    for (int64_t f = 0; f < q->N; ++f) cr[f] += qv * wr[f];
  }
  q->d1[row] = amax;
}

void rfo_quant_gemm(const double* a, const double* w, int64_t M, int64_t K, int64_t N,
                    double fmax, double* d1, double* c, int threads) {
  quant_ctx q = {a, w, K, N, 0, fmax, d1, c};
  for_rows(quant_row, &q, M, threads);
}

/* Smallest power of two >= x (x > 0); 0 for x == 0. */
static float pow2_ceil(float x) {
  if (!(x > 0.0f)) return 0.0f;
  int e;
  float f = frexpf(x, &e); /* x = f 2^e, f in [0.5, 1) */
  return f == 0.5f ? ldexpf(1.0f, e - 1) : ldexpf(1.0f, e);
}

static void quant_e4m3_row(void* vctx, int64_t row) {
  quant_ctx* q = (quant_ctx*)vctx;
  const double* ar = q->a + row * q->K;
  double* cr = q->c + row * q->N;
  for (int64_t f = 0; f < q->N; ++f) cr[f] = 0.0;
  float amax = 0.0f; /* running d1 (float32, as the kernel keeps it) */
  float ref = 0.0f;  /* H' reference: power of two >= running d1 */
  int64_t tk = q->tile_k > 0 ? q->tile_k : q->K;
  for (int64_t l0 = 0; l0 < q->K; l0 += tk) {
    int64_t l1 = l0 + tk < q->K ? l0 + tk : q->K;
    for (int64_t l = l0; l < l1; ++l) amax = fmaxf(amax, fabsf((float)ar[l]));
    float nref = pow2_ceil(amax);
    /* Eq.17 correction of the accumulator, corr = H'(d1')/H'(d1) = ref'/ref
     * (quant_gemm d2: d1'/d1 with d1 replaced by its power-of-two H' proxy) */
    if (l0 > 0 && nref != ref && ref > 0.0f) {
      double corr = (double)ref / (double)nref;
      for (int64_t f = 0; f < q->N; ++f) cr[f] *= corr;
    }
    ref = nref;
    /* exact: fmax * 2^-e; while the running absmax is 0 every element so far is
     * 0 and the guarded H' is the identity (the reference's repair): the tile
     * contributes 0 (a scale of fmax / 0 would turn 0 * inf into NaN) */
    float scale = ref > 0.0f ? (float)q->fmax / ref : 0.0f;
    for (int64_t l = l0; l < l1; ++l) {
      double qv = (double)rfo_round_e4m3((float)ar[l] * scale);
      const double* wr = q->w + l * q->N;
      for (int64_t f = 0; f < q->N; ++f) cr[f] += qv * wr[f];
    }
  }
  /* finalize_root: retarget H'(ref) -> H(d1): c *= ref / d1 (0/0 -> NaN) */
  double fin = (double)ref / (double)amax;
  for (int64_t f = 0; f < q->N; ++f) cr[f] *= fin;
  q->d1[row] = amax;
}

void rfo_quant_gemm_e4m3(const double* a, const double* w, int64_t M, int64_t K, int64_t N,
                         double fmax, int64_t tile_k, double* d1, double* c, int threads) {
  quant_ctx q = {a, w, K, N, tile_k, fmax, d1, c};
  for_rows(quant_e4m3_row, &q, M, threads);
}

/* ----------------------------------------------------------- rmsnorm --- */

typedef struct {
  const double *x, *g, *w;
  int64_t K, N;
  double eps;
  double *d1, *y;
} rms_ctx;

static void rms_row(void* vctx, int64_t row) {
  rms_ctx* c = (rms_ctx*)vctx;
  const double* xr = c->x + row * c->K;
  double ss = 0;
  for (int64_t l = 0; l < c->K; ++l) ss += xr[l] * xr[l];
  double den = sqrt(ss * (1.0 / (double)c->K) + c->eps);
  double* yr = c->y + row * c->N;
  for (int64_t f = 0; f < c->N; ++f) yr[f] = 0.0;
  for (int64_t l = 0; l < c->K; ++l) {
    double s = xr[l] * c->g[l] / den;
    const double* wr = c->w + l * c->N;
    for (int64_t f = 0; f < c->N; ++f) yr[f] += s * wr[f];
  }
  c->d1[row] = ss;
}

void rfo_rmsnorm_gemm(const double* x, const double* g, const double* w, int64_t T,
                      int64_t K, int64_t N, double eps, double* d1, double* y, int threads) {
  rms_ctx c = {x, g, w, K, N, eps, d1, y};
  for_rows(rms_row, &c, T, threads);
}

void rfo_rmsnorm_gemm_incremental(const double* x, const double* g, const double* w,
                                  int64_t K, int64_t N, double eps, double* d1,
                                  double* y) {
  double invk = 1.0 / (double)K;
  double ss = 0.0;
  for (int64_t f = 0; f < N; ++f) y[f] = 0.0;
  for (int64_t l = 0; l < K; ++l) {
    double prev = ss;
    ss += x[l] * x[l];
    if (l > 0) { /* corr = sqrt(INVK*d1' + EPS)/sqrt(INVK*d1 + EPS) */
      double corr = sqrt(invk * prev + eps) / sqrt(invk * ss + eps);
      for (int64_t f = 0; f < N; ++f) y[f] *= corr;
    }
    double s = x[l] * g[l] / sqrt(ss * invk + eps);
    for (int64_t f = 0; f < N; ++f) y[f] += s * w[l * N + f];
  }
  *d1 = ss;
}

/* --------------------------------------------------------- layernorm --- */

typedef struct {
  const double *x, *g, *w;
  int64_t K, N;
  double eps;
  double *d1, *d2, *d3, *d4;
} ln_ctx;

/* run_unfused order (simulator.cpp:377-421): d1, d2 over the whole row, then
 * d3[f] = sum x g w / sigma and d4[f] = sum (d1/K) g w / sigma with
 * sigma = sqrt(d2/K - (d1/K)^2 + eps), exactly the DSL's expression tree. */
static void ln_row(void* vctx, int64_t row) {
  ln_ctx* c = (ln_ctx*)vctx;
  const double* xr = c->x + row * c->K;
  const double invk = 1.0 / (double)c->K;
  double s1 = 0, s2 = 0;
  for (int64_t l = 0; l < c->K; ++l) s1 += xr[l];
  for (int64_t l = 0; l < c->K; ++l) s2 += xr[l] * xr[l];
  double sig = sqrt(s2 * invk - s1 * invk * s1 * invk + c->eps);
  double* y3 = c->d3 + row * c->N;
  double* y4 = c->d4 + row * c->N;
  for (int64_t f = 0; f < c->N; ++f) y3[f] = y4[f] = 0.0;
  for (int64_t l = 0; l < c->K; ++l) {
    double a3 = xr[l] * c->g[l] / sig;
    double a4 = s1 * invk * c->g[l] / sig;
    const double* wr = c->w + l * c->N;
    for (int64_t f = 0; f < c->N; ++f) {
      y3[f] += a3 * wr[f];
      y4[f] += a4 * wr[f];
    }
  }
  c->d1[row] = s1;
  c->d2[row] = s2;
}

void rfo_layernorm_gemm(const double* x, const double* g, const double* w, int64_t T,
                        int64_t K, int64_t N, double eps, double* d1, double* d2, double* d3,
                        double* d4, int threads) {
  ln_ctx c = {x, g, w, K, N, eps, d1, d2, d3, d4};
  for_rows(ln_row, &c, T, threads);
}

void rfo_layernorm_gemm_incremental(const double* x, const double* g, const double* w,
                                    int64_t K, int64_t N, double eps, double* d1, double* d2,
                                    double* d3, double* d4) {
  const double invk = 1.0 / (double)K;
  double s1 = 0, s2 = 0;
  for (int64_t f = 0; f < N; ++f) d3[f] = d4[f] = 0.0;
  for (int64_t l = 0; l < K; ++l) {
    double p1 = s1, p2 = s2;
    s1 += x[l];
    s2 += x[l] * x[l];
    double sig = sqrt(s2 * invk - s1 * invk * s1 * invk + eps);
    if (l > 0) { /* corr3 = sigma'/sigma; corr4 = (d1/d1') * sigma'/sigma */
      double sigp = sqrt(p2 * invk - p1 * invk * p1 * invk + eps);
      double c3 = sigp / sig, c4 = (s1 / p1) * sigp / sig;
      for (int64_t f = 0; f < N; ++f) {
        d3[f] *= c3;
        d4[f] *= c4;
      }
    }
    double a3 = x[l] * g[l] / sig, a4 = s1 * invk * g[l] / sig;
    for (int64_t f = 0; f < N; ++f) {
      d3[f] += a3 * w[l * N + f];
      d4[f] += a4 * w[l * N + f];
    }
  }
  *d1 = s1;
  *d2 = s2;
}

/* ------------------------------------------------------ row statistics --- */

/* make_variance's oracle (workloads.cpp:246-277), per row */
void rfo_variance(const double* x, int64_t rows, int64_t n, double* d1, double* d2) {
  for (int64_t r = 0; r < rows; ++r) {
    double s = 0, q = 0;
    for (int64_t i = 0; i < n; ++i) {
      s += x[r * n + i];
      q += x[r * n + i] * x[r * n + i];
    }
    d1[r] = s;
    d2[r] = q;
  }
}

/* make_sum_sum's oracle (workloads.cpp:213-242): d2 = sum x1 x2 / sqrt(max(d1 - c, eps)) */
void rfo_sum_sum(const double* x1, const double* x2, int64_t rows, int64_t n, double c,
                 double eps, double* d1, double* d2) {
  for (int64_t r = 0; r < rows; ++r) {
    double m = 0, s = 0;
    for (int64_t i = 0; i < n; ++i) m += x1[r * n + i] * x1[r * n + i];
    const double den = sqrt(fmax(m - c, eps));
    for (int64_t i = 0; i < n; ++i) s += x1[r * n + i] * x2[r * n + i] / den;
    d1[r] = m;
    d2[r] = s;
  }
}

/* moment_of_inertia's oracle (workloads.cpp:280-331), F position lanes */
void rfo_moments(const double* mass, const double* pos, int64_t rows, int64_t n, int64_t F,
                 double* d1, double* d2, double* d3) {
  for (int64_t r = 0; r < rows; ++r) {
    const double* m = mass + r * n;
    const double* p = pos + r * n * F;
    double t = 0;
    for (int64_t l = 0; l < n; ++l) t += m[l];
    d1[r] = t;
    for (int64_t f = 0; f < F; ++f) d2[r * F + f] = d3[r * F + f] = 0.0;
    for (int64_t l = 0; l < n; ++l)
      for (int64_t f = 0; f < F; ++f) {
        d2[r * F + f] += m[l] * p[l * F + f];
        d3[r * F + f] += m[l] * p[l * F + f] * p[l * F + f];
      }
  }
}

/* --------------------------------------------------------- moe routing --- */

void rfo_moe_routing(const double* s, int64_t rows, int64_t experts, int64_t k,
                     double* d1, double* d2, double* topk_val, int64_t* topk_idx) {
  int64_t kk = k < experts ? k : experts;
  for (int64_t r = 0; r < rows; ++r) {
    const double* sr = s + r * experts;
    double m = sr[0];
    for (int64_t i = 0; i < experts; ++i) m = fmax(m, sr[i]);
    double t = 0;
    for (int64_t i = 0; i < experts; ++i) t += exp(sr[i] - m);
    d1[r] = m;
    d2[r] = t;
    /* selection: descending value, ties to the lowest index */
    for (int64_t j = 0; j < kk; ++j) {
      int64_t best = -1;
      for (int64_t i = 0; i < experts; ++i) {
        int taken = 0;
        for (int64_t u = 0; u < j; ++u)
          if (topk_idx[r * k + u] == i + 1) taken = 1;
        if (taken) continue;
        if (best < 0 || sr[i] > sr[best]) best = i;
      }
      topk_val[r * k + j] = sr[best];
      topk_idx[r * k + j] = best + 1;
    }
  }
}

/* -------------------------------------------------------------- parity --- */

/* ---------------------------------------------------------- run_fused --- */

/* One partial state: d1, d2 scalars and d3 [hd] (attention). */
typedef struct {
  double d1, d2;
  double* d3;
} fstate;

/* Correction of reduction idx (2 or 3) from the child's dependency values to
 * the target's: retarget_factor (simulator.cpp:278-318) for each pattern's H. */
static double fused_factor(int pattern, int idx, const fstate* from, double t1, double t2, double c,
                           double eps) {
  switch (pattern) {
    case 1: return exp(from->d1 - t1);                                   /* e^(d1'-d1) */
    case 2: return idx == 2 ? exp(from->d1 - t1) : exp(from->d1 - t1) * from->d2 / t2;
    case 8: return sqrt(fmax(from->d1 - c, eps)) / sqrt(fmax(t1 - c, eps));
    default: return 1.0; /* variance: no dependency */
  }
}

int rfo_fused_row(int pattern, const double* a, const double* b, int64_t hd, const int64_t* levels,
                  int depth, int k, double c, double eps, double* d1, double* d2, double* d3) {
  if (depth < 1 || k < 1 || k > depth || levels[depth] != 1) return -1;
  for (int m = 1; m <= depth; ++m)
    if (levels[m] < 1 || levels[m - 1] % levels[m]) return -1;
  const int64_t n1 = levels[1], seg = levels[0] / n1;
  const int att = pattern == 2;
  fstate* cur = calloc((size_t)n1, sizeof(fstate));
  double* o1 = att ? calloc((size_t)(n1 * hd), sizeof(double)) : NULL;
  /* level 1: buffered segments, reductions in dependency order */
  for (int64_t j = 0; j < n1; ++j) {
    const double* x = a + j * seg;
    fstate* s = &cur[j];
    s->d3 = att ? o1 + j * hd : NULL;
    if (pattern == 1 || att) {
      s->d1 = -INFINITY;
      for (int64_t l = 0; l < seg; ++l) s->d1 = fmax(s->d1, x[l]);
      for (int64_t l = 0; l < seg; ++l) s->d2 += exp(x[l] - s->d1);
      if (att)
        for (int64_t l = 0; l < seg; ++l) {
          const double w = exp(x[l] - s->d1) / s->d2;
          for (int64_t f = 0; f < hd; ++f) s->d3[f] += w * b[(j * seg + l) * hd + f];
        }
    } else if (pattern == 7) {
      for (int64_t l = 0; l < seg; ++l) s->d1 += x[l];
      for (int64_t l = 0; l < seg; ++l) s->d2 += x[l] * x[l];
    } else {
      for (int64_t l = 0; l < seg; ++l) s->d1 += x[l] * x[l];
      const double h = sqrt(fmax(s->d1 - c, eps));
      for (int64_t l = 0; l < seg; ++l) s->d2 += x[l] * b[j * seg + l] / h;
    }
  }
  /* levels 2..k: group combines, children corrected to the group's values */
  int64_t width = n1;
  for (int m = 2; m <= k; ++m) {
    const int64_t w2 = levels[m], group = width / w2;
    for (int64_t j = 0; j < w2; ++j) {
      fstate g = {(pattern == 1 || att) ? -INFINITY : 0.0, 0.0, NULL};
      double og[hd > 0 ? hd : 1];
      memset(og, 0, sizeof og);
      for (int64_t q = 0; q < group; ++q) { /* reduction 1: plain */
        const fstate* ch = &cur[j * group + q];
        g.d1 = (pattern == 1 || att) ? fmax(g.d1, ch->d1) : g.d1 + ch->d1;
      }
      for (int64_t q = 0; q < group; ++q) /* reduction 2: corrected to g.d1 */
        g.d2 += cur[j * group + q].d2 * fused_factor(pattern, 2, &cur[j * group + q], g.d1, 0, c, eps);
      if (att)
        for (int64_t q = 0; q < group; ++q) { /* reduction 3: corrected to (g.d1, g.d2) */
          const fstate* ch = &cur[j * group + q];
          const double f = fused_factor(pattern, 3, ch, g.d1, g.d2, c, eps);
          for (int64_t e = 0; e < hd; ++e) og[e] += ch->d3[e] * f;
        }
      cur[j].d1 = g.d1;
      cur[j].d2 = g.d2;
      if (att) memcpy(cur[j].d3, og, sizeof(double) * (size_t)hd);
    }
    width = w2;
  }
  /* bridge + plain fold above level k, reduction by reduction */
  double f1 = (pattern == 1 || att) ? -INFINITY : 0.0, f2 = 0.0;
  for (int64_t j = 0; j < width; ++j) f1 = (pattern == 1 || att) ? fmax(f1, cur[j].d1) : f1 + cur[j].d1;
  for (int64_t j = 0; j < width; ++j) f2 += cur[j].d2 * fused_factor(pattern, 2, &cur[j], f1, 0, c, eps);
  *d1 = f1;
  *d2 = f2;
  if (att) {
    for (int64_t e = 0; e < hd; ++e) d3[e] = 0.0;
    for (int64_t j = 0; j < width; ++j) {
      const double f = fused_factor(pattern, 3, &cur[j], f1, f2, c, eps);
      for (int64_t e = 0; e < hd; ++e) d3[e] += cur[j].d3[e] * f;
    }
  }
  free(o1);
  free(cur);
  return 0;
}

double rfo_scaled_max_err(const double* x, const double* y, int64_t n, int64_t* worst) {
  double mx = 0.0;
  int64_t wi = -1;
  for (int64_t i = 0; i < n; ++i) {
    double a = x[i], b = y[i], e;
    if (a == b) e = 0.0;
    else if (isnan(a) || isnan(b) || isinf(a) || isinf(b)) e = INFINITY;
    else e = fabs(a - b) / (1.0 + fmax(fabs(a), fabs(b)));
    if (e > mx || (wi < 0 && e > 0)) {
      mx = e;
      wi = i;
    }
  }
  if (worst) *worst = wi;
  return mx;
}
