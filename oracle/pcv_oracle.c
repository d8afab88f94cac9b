/*
 * TEST INFRASTRUCTURE ONLY - CPU oracle for the PCV hot path. See pcv_oracle.h.
 * Plain C restatement of /root/reference/proj; each function cites what it follows.
 * Compiled without FMA contraction (baseline x86-64, -ffp-contract=off) like the reference's
 * Release build, so that same-order arithmetic reproduces the reference bit for bit.
 */
#define _GNU_SOURCE
#include "pcv_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

static __thread char g_err[512];
const char* pcvo_last_error(void) { return g_err; }
static int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------------ math.hpp:17-109 */
#define NEG_INF (-INFINITY)
static const double kLog2Pi = 1.8378770664093454835606594728112;

static double logaddexp(double a, double b) { /* math.hpp:17-22 */
  if (a == NEG_INF) return b;
  if (b == NEG_INF) return a;
  const double m = a > b ? a : b;
  return m + log1p(exp(-fabs(a - b)));
}
static double logsumexp(const double* v, int n) { /* math.hpp:24-32 */
  double m = NEG_INF;
  for (int i = 0; i < n; ++i)
    if (v[i] > m) m = v[i];
  if (m == NEG_INF) return NEG_INF;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += exp(v[i] - m);
  return m + log(s);
}
static double normal_cdf(double z) { return 0.5 * erfc(-z * 0.70710678118654752440084436210485); }
static double normal_logpdf(double x, double mean, double var) { /* math.hpp:39-42 */
  const double r = x - mean;
  return -0.5 * (kLog2Pi + log(var) + r * r / var);
}
/* math.hpp:94-109 */
static double mvn_logpdf_compound(const double* x, const double* mean, int n, double sigma2,
                                  double tau2) {
  if (!(sigma2 > 0.0) || tau2 < 0.0) return NEG_INF;
  double ss = 0.0, sr = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = x[i] - mean[i];
    ss += r * r;
    sr += r;
  }
  const double denom = sigma2 + n * tau2;
  const double quad = (ss - tau2 * sr * sr / denom) / sigma2;
  const double logdet = (n - 1) * log(sigma2) + log(denom);
  return -0.5 * (n * kLog2Pi + logdet + quad);
}
/* priors.hpp:13-26 */
static double log_half_normal(double x, double v) {
  return 0.5 * log(2.0 / (3.141592653589793238462643383279 * v)) - x * x / (2.0 * v);
}
static double log_gamma_pdf(double x, double a, double r) {
  return a * log(r) - lgamma(a) + (a - 1.0) * log(x) - r * x;
}
static double log_beta_pdf(double x, double a, double b) {
  return (a - 1.0) * log(x) + (b - 1.0) * log1p(-x) + lgamma(a + b) - lgamma(a) - lgamma(b);
}

/* ------------------------------------------------------------------ rng.hpp:18-143 */
static uint64_t mix64(uint64_t z) { /* rng.hpp:18-23 */
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t pcvo_stream_key(uint64_t kind, uint64_t a, uint64_t b, uint64_t c) { /* rng.hpp:35-43 */
  uint64_t k = mix64(kind);
  k = mix64(k ^ a);
  k = mix64(k ^ b);
  k = mix64(k ^ c);
  return k;
}
void pcvo_rng_init(pcvo_rng* r, uint64_t seed, uint64_t stream) { /* rng.hpp:49-56 */
  memset(r, 0, sizeof *r);
  r->key[0] = (uint32_t)seed;
  r->key[1] = (uint32_t)(seed >> 32);
  r->ctr[2] = (uint32_t)stream;
  r->ctr[3] = (uint32_t)(stream >> 32);
}
static void refill(pcvo_rng* r) { /* rng.hpp:115-135: Philox4x32-10 */
  uint32_t c0 = r->ctr[0], c1 = r->ctr[1], c2 = r->ctr[2], c3 = r->ctr[3];
  uint32_t k0 = r->key[0], k1 = r->key[1];
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32);
    const uint32_t lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  r->buf[0] = c0;
  r->buf[1] = c1;
  r->buf[2] = c2;
  r->buf[3] = c3;
  r->have = 4;
  if (++r->ctr[0] == 0) ++r->ctr[1];
}
uint32_t pcvo_next_u32(pcvo_rng* r) { /* rng.hpp:58-61 */
  if (r->have == 0) refill(r);
  return r->buf[4 - r->have--];
}
uint64_t pcvo_next_u64(pcvo_rng* r) { /* rng.hpp:63-67 */
  const uint64_t lo = pcvo_next_u32(r);
  const uint64_t hi = pcvo_next_u32(r);
  return lo | (hi << 32);
}
double pcvo_uniform(pcvo_rng* r) { /* rng.hpp:70-72 */
  return ((double)(pcvo_next_u64(r) >> 11) + 0.5) * 0x1p-53;
}
double pcvo_normal(pcvo_rng* r) { /* rng.hpp:75-87: Box-Muller with cached second variate */
  if (r->has_cached) {
    r->has_cached = 0;
    return r->cached;
  }
  const double u1 = pcvo_uniform(r);
  const double u2 = pcvo_uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  r->cached = rad * sin(a);
  r->has_cached = 1;
  return rad * cos(a);
}
void pcvo_skip_to(pcvo_rng* r, uint64_t block) { /* rng.hpp:91-96 */
  r->ctr[0] = (uint32_t)block;
  r->ctr[1] = (uint32_t)(block >> 32);
  r->have = 0;
  r->has_cached = 0;
}
uint64_t pcvo_below(pcvo_rng* r, uint64_t n) { /* rng.hpp:99-105 */
  const uint64_t bound = n * ((~(uint64_t)0) / n);
  for (;;) {
    const uint64_t v = pcvo_next_u64(r);
    if (v < bound) return v % n;
  }
}
int pcvo_rng_sequence(uint64_t seed, uint64_t stream, int32_t do_skip, uint64_t skip_block,
                      const char* ops, const uint64_t* arg, int64_t n, double* out) {
  pcvo_rng r;
  pcvo_rng_init(&r, seed, stream);
  if (do_skip) pcvo_skip_to(&r, skip_block);
  for (int64_t i = 0; i < n; ++i) {
    switch (ops[i]) {
      case 'u': out[i] = pcvo_uniform(&r); break;
      case 'n': out[i] = pcvo_normal(&r); break;
      case '4': out[i] = (double)pcvo_next_u32(&r); break;
      case 'b': out[i] = (double)pcvo_below(&r, arg[i]); break;
      default: return set_err(PCVG_INVALID_INPUT, "bad rng op");
    }
  }
  return 0;
}

/* ------------------------------------------------------------------ folds.cpp:43-108 */
int pcvo_make_kfold(int64_t n, int32_t K, uint64_t seed, int32_t* out) { /* folds.cpp:65-84 */
  if (K < 2 || K > n) return set_err(PCVG_INVALID_INPUT, "K-fold requires 2 <= K <= n_obs");
  const int64_t base = n / K, rem = n % K;
  int64_t pos = 0;
  for (int k = 0; k < K; ++k)
    for (int64_t i = 0; i < base + (k < rem ? 1 : 0); ++i) out[pos++] = k;
  pcvo_rng r;
  pcvo_rng_init(&r, seed, pcvo_stream_key(PCVG_STREAM_KFOLD, (uint64_t)K, 0, 0));
  for (int64_t i = n - 1; i > 0; --i) {
    const int64_t j = (int64_t)pcvo_below(&r, (uint64_t)(i + 1));
    const int32_t t = out[i];
    out[i] = out[j];
    out[j] = t;
  }
  return 0;
}

/* Stable argsort by time (std::stable_sort in folds.cpp:95-98), merge sort. */
/* cfg2 logistic simulator (new family; same draw order as oracle/ref_shim.cpp
 * pcvref_simulate_logistic on the reference CounterRng). */
int pcvo_simulate_logistic(int64_t n, int32_t P, uint64_t seed, double* y, double* x) {
  if (n < 2 || P < 1) return set_err(PCVG_INVALID_INPUT, "logistic simulator needs n >= 2, P >= 1");
  pcvo_rng rng;
  pcvo_rng_init(&rng, seed, pcvo_stream_key(PCVG_STREAM_SIMULATE, 5, 0, 0));
  double* beta = (double*)malloc(sizeof(double) * (size_t)(P + 1));
  for (int32_t j = 0; j <= P; ++j) beta[j] = pcvo_normal(&rng);
  const double scale = 1.0 / sqrt((double)P);
  for (int64_t i = 0; i < n; ++i) {
    double eta = beta[0];
    for (int32_t j = 0; j < P; ++j) {
      x[i * P + j] = pcvo_normal(&rng) * scale;
      eta += x[i * P + j] * beta[1 + j];
    }
    y[i] = pcvo_uniform(&rng) < 1.0 / (1.0 + exp(-eta)) ? 1.0 : 0.0;
  }
  free(beta);
  return 0;
}

static void time_order(const int64_t* t, int64_t n, int64_t* order) {
  int64_t* tmp = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  for (int64_t w = 1; w < n; w *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * w) {
      int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
      int64_t a = lo, b = mid, o = lo;
      while (a < mid && b < hi) tmp[o++] = (t[order[b]] < t[order[a]]) ? order[b++] : order[a++];
      while (a < mid) tmp[o++] = order[a++];
      while (b < hi) tmp[o++] = order[b++];
    }
    memcpy(order, tmp, sizeof(int64_t) * n);
  }
  free(tmp);
}

int pcvo_make_time_blocks(const pcvg_dataset* d, int32_t K, int32_t* out) { /* folds.cpp:86-108 */
  const int64_t n = d->n_obs;
  if (!d->time_index) return set_err(PCVG_INVALID_INPUT, "time-block scheme requires a time column");
  if (K < 2 || K > n) return set_err(PCVG_INVALID_INPUT, "time-block scheme requires 2 <= K <= n_obs");
  int64_t* order = malloc(sizeof(int64_t) * n);
  time_order(d->time_index, n, order);
  const int64_t base = n / K, rem = n % K;
  int64_t pos = 0;
  for (int k = 0; k < K; ++k) {
    const int64_t len = base + (k < rem ? 1 : 0);
    for (int64_t i = 0; i < len; ++i) out[order[pos++]] = k;
  }
  free(order);
  return 0;
}

/* hv-block (new, unpinned by the reference: SPEC.md:114). Test blocks are the time-block
 * partition (folds.cpp:99-106 sizes); training drops h ranks on each side of the block. */
int pcvo_make_hv_block(const pcvg_dataset* d, int32_t K, int64_t h, int64_t* iv) {
  const int64_t n = d->n_obs;
  if (!d->time_index) return set_err(PCVG_INVALID_INPUT, "hv-block requires a time column");
  if (K < 2 || K > n || h < 0) return set_err(PCVG_INVALID_INPUT, "hv-block requires 2 <= K <= n_obs, h >= 0");
  const int64_t base = n / K, rem = n % K;
  int64_t pos = 0;
  for (int k = 0; k < K; ++k) {
    const int64_t len = base + (k < rem ? 1 : 0);
    const int64_t lo = pos, hi = pos + len;
    iv[4 * k] = lo;
    iv[4 * k + 1] = hi;
    iv[4 * k + 2] = lo - h < 0 ? 0 : lo - h;
    iv[4 * k + 3] = hi + h > n ? n : hi + h;
    if (iv[4 * k + 3] - iv[4 * k + 2] >= n) return set_err(PCVG_INVALID_INPUT, "hv-block fold has empty training set");
    pos = hi;
  }
  return 0;
}

int pcvo_make_hv_racine(const pcvg_dataset* d, int64_t v, int64_t h, int64_t* iv) {
  const int64_t n = d->n_obs;
  if (!d->time_index) return set_err(PCVG_INVALID_INPUT, "hv-block requires a time column");
  if (v < 0 || h < 0) return set_err(PCVG_INVALID_INPUT, "hv-block requires v, h >= 0");
  for (int64_t t = 0; t < n; ++t) {
    int64_t lo = t - v < 0 ? 0 : t - v, hi = t + v + 1 > n ? n : t + v + 1;
    int64_t elo = t - v - h < 0 ? 0 : t - v - h, ehi = t + v + h + 1 > n ? n : t + v + h + 1;
    if (ehi - elo >= n) return set_err(PCVG_INVALID_INPUT, "hv-block fold has empty training set");
    iv[4 * t] = lo;
    iv[4 * t + 1] = hi;
    iv[4 * t + 2] = elo;
    iv[4 * t + 3] = ehi;
  }
  return 0;
}

/* ------------------------------------------------------------------ models */
struct pcvo_model {
  int family;
  int broken_fold; /* test_engine.cpp:57-90 BrokenFoldModel: gradient NaN on this fold (-1 = none) */
  int64_t n;
  int ncov;
  double *y, *x;
  int32_t* g;
  int64_t* rank; /* time rank (hv folds) */
  int K;
  int32_t* test_index; /* partition or NULL */
  int64_t* iv;         /* hv intervals or NULL */
  int J, P, dim;
  int32_t* mask; /* grouped covariate mask */
  int include_floor, p, q, rho_sym;
  int per_subject; /* rat growth M_A (rat_growth.hpp:22-27) */
  /* per-fold test layout (fold_meta_, grouped_regression.cpp:27-47): segments of test rows
   * grouped by group in increasing group order, rows increasing within a group. */
  int64_t* fold_seg; /* [K+1] */
  int32_t* seg_group;
  int32_t* seg_unseen;
  int64_t* seg_row; /* [nseg+1] */
  int32_t* rows;
};

static int excluded(const pcvo_model* m, int64_t i, int fold) { /* not a training row */
  if (fold >= m->K) return 0;
  if (m->test_index) return m->test_index[i] == fold;
  const int64_t r = m->rank[i];
  return r >= m->iv[4 * fold + 2] && r < m->iv[4 * fold + 3];
}
static int in_test(const pcvo_model* m, int64_t i, int fold) {
  if (fold >= m->K) return 0;
  if (m->test_index) return m->test_index[i] == fold;
  const int64_t r = m->rank[i];
  return r >= m->iv[4 * fold] && r < m->iv[4 * fold + 1];
}

void pcvo_model_destroy(pcvo_model* m) {
  if (!m) return;
  free(m->y); free(m->x); free(m->g); free(m->rank); free(m->test_index); free(m->iv);
  free(m->mask); free(m->fold_seg); free(m->seg_group); free(m->seg_unseen); free(m->seg_row);
  free(m->rows);
  free(m);
}

pcvo_model* pcvo_model_create(const pcvg_dataset* d, const pcvg_folds* f,
                              const pcvg_model_spec* s) {
  pcvo_model* m = calloc(1, sizeof *m);
  m->broken_fold = -1;
  const int64_t n = d->n_obs;
  m->family = s->family;
  m->n = n;
  m->ncov = d->n_cov;
  m->K = f->K;
  m->y = malloc(sizeof(double) * n);
  memcpy(m->y, d->y, sizeof(double) * n);
  m->x = malloc(sizeof(double) * (n * d->n_cov + 1));
  if (d->n_cov) memcpy(m->x, d->x, sizeof(double) * n * d->n_cov);
  m->J = 0;
  if (d->group_id) {
    m->g = malloc(sizeof(int32_t) * n);
    memcpy(m->g, d->group_id, sizeof(int32_t) * n);
    for (int64_t i = 0; i < n; ++i)
      if (m->g[i] + 1 > m->J) m->J = m->g[i] + 1;
  }
  if (f->test_index) {
    m->test_index = malloc(sizeof(int32_t) * n);
    memcpy(m->test_index, f->test_index, sizeof(int32_t) * n);
  } else {
    if (!d->time_index) { set_err(PCVG_INVALID_INPUT, "hv-block needs time"); pcvo_model_destroy(m); return NULL; }
    m->iv = malloc(sizeof(int64_t) * 4 * f->K);
    memcpy(m->iv, f->intervals, sizeof(int64_t) * 4 * f->K);
    int64_t* order = malloc(sizeof(int64_t) * n);
    time_order(d->time_index, n, order);
    m->rank = malloc(sizeof(int64_t) * n);
    for (int64_t r = 0; r < n; ++r) m->rank[order[r]] = r;
    free(order);
  }
  switch (s->family) {
    case PCVG_FAMILY_GROUPED:
      if (!m->g) { set_err(PCVG_INVALID_INPUT, "grouped regression needs a group column"); pcvo_model_destroy(m); return NULL; }
      m->P = d->n_cov;
      m->mask = malloc(sizeof(int32_t) * (m->P + 1));
      for (int p = 0; p < m->P; ++p) m->mask[p] = s->covariate_mask ? s->covariate_mask[p] : 1;
      m->dim = m->J + m->P + 3;
      break;
    case PCVG_FAMILY_RADON:
      if (!m->g || d->n_cov < 1) { set_err(PCVG_INVALID_INPUT, "radon needs groups and a floor covariate"); pcvo_model_destroy(m); return NULL; }
      m->include_floor = s->include_floor != 0;
      m->dim = m->J + 4;
      break;
    case PCVG_FAMILY_SEASONAL_AR:
      m->p = s->ar_order;
      m->q = s->dummies;
      m->rho_sym = s->rho_transform == PCVG_RHO_SYMMETRIC;
      if (m->p < 1 || m->q < 0 || d->n_cov < m->p + m->q) { set_err(PCVG_INVALID_INPUT, "bad seasonal spec"); pcvo_model_destroy(m); return NULL; }
      m->dim = m->p + m->q + 2;
      m->J = 0;
      break;
    case PCVG_FAMILY_LOGISTIC:
      m->P = d->n_cov;
      m->dim = m->P + 1;
      m->J = 0;
      break;
    case PCVG_FAMILY_RAT_GROWTH: /* rat_growth.cpp:13-48 */
      if (!m->g || d->n_cov < 1) { set_err(PCVG_INVALID_INPUT, "growth model needs a group column and a time covariate"); pcvo_model_destroy(m); return NULL; }
      m->per_subject = s->per_subject_slope != 0;
      m->dim = m->per_subject ? 2 * m->J + 5 : m->J + 4;
      break;
    default:
      set_err(PCVG_INVALID_INPUT, "family not in the oracle");
      pcvo_model_destroy(m);
      return NULL;
  }
  /* Per-fold test segments. */
  const int K = m->K;
  const int hier = (m->family == PCVG_FAMILY_GROUPED || m->family == PCVG_FAMILY_RADON ||
                    m->family == PCVG_FAMILY_RAT_GROWTH);
  const int J = hier ? m->J : 1;
  int64_t* grp_size = calloc(J, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) grp_size[hier ? m->g[i] : 0]++;
  int64_t cap_seg = 16, cap_rows = n + 16, nseg = 0, nrows = 0;
  m->fold_seg = malloc(sizeof(int64_t) * (K + 1));
  m->seg_group = malloc(sizeof(int32_t) * cap_seg);
  m->seg_unseen = malloc(sizeof(int32_t) * cap_seg);
  m->seg_row = malloc(sizeof(int64_t) * (cap_seg + 1));
  m->rows = malloc(sizeof(int32_t) * cap_rows);
  int64_t* excl = calloc(J, sizeof(int64_t));
  int64_t* cnt = calloc(J, sizeof(int64_t));
  int64_t* start = calloc(J, sizeof(int64_t));
  int32_t* tmp = malloc(sizeof(int32_t) * (n + 1));
  /* bucket test rows per fold for partitions */
  int64_t* part_ptr = NULL;
  int32_t* part_rows = NULL;
  if (m->test_index) {
    part_ptr = calloc(K + 1, sizeof(int64_t));
    part_rows = malloc(sizeof(int32_t) * n);
    for (int64_t i = 0; i < n; ++i) part_ptr[m->test_index[i] + 1]++;
    for (int k = 0; k < K; ++k) part_ptr[k + 1] += part_ptr[k];
    int64_t* fill = malloc(sizeof(int64_t) * (K + 1));
    memcpy(fill, part_ptr, sizeof(int64_t) * (K + 1));
    for (int64_t i = 0; i < n; ++i) part_rows[fill[m->test_index[i]]++] = (int32_t)i;
    free(fill);
  }
  for (int k = 0; k < K; ++k) {
    m->fold_seg[k] = nseg;
    /* test rows of fold k in row order */
    int64_t nt = 0;
    if (m->test_index) {
      for (int64_t t = part_ptr[k]; t < part_ptr[k + 1]; ++t) tmp[nt++] = part_rows[t];
    } else {
      for (int64_t i = 0; i < n; ++i)
        if (in_test(m, i, k)) tmp[nt++] = (int32_t)i;
    }
    memset(excl, 0, sizeof(int64_t) * J);
    memset(cnt, 0, sizeof(int64_t) * J);
    if (m->test_index) {
      for (int64_t t = 0; t < nt; ++t) excl[hier ? m->g[tmp[t]] : 0]++;
    } else {
      for (int64_t i = 0; i < n; ++i)
        if (excluded(m, i, k)) excl[hier ? m->g[i] : 0]++;
    }
    for (int64_t t = 0; t < nt; ++t) cnt[hier ? m->g[tmp[t]] : 0]++;
    /* group-ordered segments */
    int64_t acc = 0;
    for (int gg = 0; gg < J; ++gg) { start[gg] = acc; acc += cnt[gg]; }
    if (nrows + nt > cap_rows) { cap_rows = 2 * (nrows + nt); m->rows = realloc(m->rows, sizeof(int32_t) * cap_rows); }
    for (int64_t t = 0; t < nt; ++t) {
      const int gg = hier ? m->g[tmp[t]] : 0;
      m->rows[nrows + start[gg]++] = tmp[t];
    }
    int64_t off = nrows;
    for (int gg = 0; gg < J; ++gg) {
      if (cnt[gg] == 0) continue;
      if (nseg + 1 >= cap_seg) {
        cap_seg *= 2;
        m->seg_group = realloc(m->seg_group, sizeof(int32_t) * cap_seg);
        m->seg_unseen = realloc(m->seg_unseen, sizeof(int32_t) * cap_seg);
        m->seg_row = realloc(m->seg_row, sizeof(int64_t) * (cap_seg + 1));
      }
      m->seg_group[nseg] = hier ? gg : -1;
      m->seg_unseen[nseg] = hier ? (grp_size[gg] - excl[gg] == 0) : 0;
      m->seg_row[nseg] = off;
      off += cnt[gg];
      ++nseg;
    }
    nrows += nt;
  }
  m->fold_seg[K] = nseg;
  m->seg_row[nseg] = nrows;
  free(grp_size); free(excl); free(cnt); free(start); free(tmp); free(part_ptr); free(part_rows);
  return m;
}

int32_t pcvo_model_dim(const pcvo_model* m) { return m->dim; }
int64_t pcvo_test_size(const pcvo_model* m, int32_t fold) {
  if (fold >= m->K) return 0;
  return m->seg_row[m->fold_seg[fold + 1]] - m->seg_row[m->fold_seg[fold]];
}
static double xv(const pcvo_model* m, int64_t i, int j) { return m->x[i * m->ncov + j]; }

/* grouped_regression.cpp:56-63 */
static double grouped_linpred(const pcvo_model* m, const double* th, int64_t i) {
  const double* beta = th + m->J;
  double mm = th[m->g[i]];
  for (int p = 0; p < m->P; ++p)
    if (m->mask[p]) mm += xv(m, i, p) * beta[p];
  return mm;
}
/* seasonal_ar.cpp:37-57 */
static double logistic_fn(double u) { return 1.0 / (1.0 + exp(-u)); }
static double rho_of(const pcvo_model* m, double u) {
  const double w = logistic_fn(u);
  return m->rho_sym ? 2.0 * w - 1.0 : 0.5 * (1.0 + w);
}
static double drho_du(const pcvo_model* m, double u) {
  const double w = logistic_fn(u);
  const double dw = w * (1.0 - w);
  return m->rho_sym ? 2.0 * dw : 0.5 * dw;
}
static double seasonal_mean(const pcvo_model* m, const double* th, int64_t i) {
  double mm = th[m->p];
  for (int a = 0; a < m->p; ++a) mm += rho_of(m, th[a]) * xv(m, i, a);
  for (int j = 0; j < m->q; ++j) mm += th[m->p + 1 + j] * xv(m, i, m->p + j);
  return mm;
}
/* rat_growth.cpp:50-63: layout M_A [alpha(J), beta(J), mu_a, mu_b, log s_a, log s_b, log s_y],
 * M_B [alpha(J), beta, mu_a, log s_a, log s_y] */
static int rat_mu_a(const pcvo_model* m) { return m->J + (m->per_subject ? m->J : 1); }
static double rat_mean(const pcvo_model* m, const double* th, int64_t i) {
  const int g = m->g[i];
  const double t = xv(m, i, 0);
  const double slope = m->per_subject ? th[m->J + g] : th[m->J];
  return th[g] + slope * t;
}
/* math.hpp:46-90 dense Cholesky MVN (mvn_logpdf_chol), n <= 64 */
static double mvn_logpdf_chol(const double* x, const double* mean, double* cov, int n) {
  for (int j = 0; j < n; ++j) {
    double dd = cov[j * n + j];
    for (int k = 0; k < j; ++k) dd -= cov[j * n + k] * cov[j * n + k];
    if (!(dd > 0.0) || !isfinite(dd)) return NEG_INF;
    const double l = sqrt(dd);
    cov[j * n + j] = l;
    for (int i = j + 1; i < n; ++i) {
      double sm = cov[i * n + j];
      for (int k = 0; k < j; ++k) sm -= cov[i * n + k] * cov[j * n + k];
      cov[i * n + j] = sm / l;
    }
  }
  double r[64];
  for (int i = 0; i < n; ++i) r[i] = x[i] - mean[i];
  for (int i = 0; i < n; ++i) {
    double sm = r[i];
    for (int k = 0; k < i; ++k) sm -= cov[i * n + k] * r[k];
    r[i] = sm / cov[i * n + i];
  }
  double q = 0.0, ld = 0.0;
  for (int i = 0; i < n; ++i) q += r[i] * r[i];
  for (int i = 0; i < n; ++i) ld += log(cov[i * n + i]);
  return -0.5 * (n * kLog2Pi + 2.0 * ld + q);
}

/* logistic plugin (oracle/ref_plugins.cpp) */
static double softplus(double t) { return (t > 0.0 ? t : 0.0) + log1p(exp(-fabs(t))); }
static double sigmoid(double t) {
  if (t >= 0.0) return 1.0 / (1.0 + exp(-t));
  const double e = exp(t);
  return e / (1.0 + e);
}
static double logit_eta(const pcvo_model* m, const double* th, int64_t i) {
  double t = th[0];
  for (int p = 0; p < m->P; ++p) t += xv(m, i, p) * th[1 + p];
  return t;
}

double pcvo_log_joint(const pcvo_model* m, const double* th, int32_t fold) {
  double lp = 0.0;
  const int J = m->J;
  switch (m->family) {
    case PCVG_FAMILY_GROUPED: { /* grouped_regression.cpp:65-85 */
      const int P = m->P;
      const double mu_a = th[J + P];
      const double sig_a = exp(th[J + P + 1]);
      const double sig_y = exp(th[J + P + 2]);
      const double va = sig_a * sig_a, vy = sig_y * sig_y;
      for (int64_t i = 0; i < m->n; ++i) {
        const double mask = excluded(m, i, fold) ? 0.0 : 1.0;
        lp += mask * normal_logpdf(m->y[i], grouped_linpred(m, th, i), vy);
      }
      for (int g = 0; g < J; ++g) lp += normal_logpdf(th[g], mu_a, va);
      lp += normal_logpdf(mu_a, 0.0, 1.0);
      for (int p = 0; p < P; ++p) lp += normal_logpdf(th[J + p], 0.0, 1.0);
      lp += log_half_normal(sig_a, 10.0) + th[J + P + 1];
      lp += log_half_normal(sig_y, 10.0) + th[J + P + 2];
      return lp;
    }
    case PCVG_FAMILY_RADON: { /* radon.cpp:50-74 */
      const double beta = th[J], mu_a = th[J + 1];
      const double va = exp(th[J + 2]), vy = exp(th[J + 3]);
      const double sa = sqrt(va);
      const double bmask = m->include_floor ? 1.0 : 0.0;
      for (int64_t i = 0; i < m->n; ++i) {
        const double mask = excluded(m, i, fold) ? 0.0 : 1.0;
        const double mean = mu_a + sa * th[m->g[i]] + bmask * beta * xv(m, i, 0);
        lp += mask * normal_logpdf(m->y[i], mean, vy);
      }
      for (int g = 0; g < J; ++g) lp += normal_logpdf(th[g], 0.0, 1.0);
      lp += normal_logpdf(beta, 0.0, 1.0);
      lp += normal_logpdf(mu_a, 0.0, 4.0);
      lp += log_gamma_pdf(va, 6.0, 9.0) + th[J + 2];
      lp += log_gamma_pdf(vy, 10.0, 10.0) + th[J + 3];
      return lp;
    }
    case PCVG_FAMILY_SEASONAL_AR: { /* seasonal_ar.cpp:59-77 */
      const int p = m->p, q = m->q;
      const double sigma = exp(th[p + q + 1]);
      const double v = sigma * sigma;
      for (int64_t i = 0; i < m->n; ++i) {
        const double mask = excluded(m, i, fold) ? 0.0 : 1.0;
        lp += mask * normal_logpdf(m->y[i], seasonal_mean(m, th, i), v);
      }
      for (int a = 0; a < p; ++a) {
        const double w = logistic_fn(th[a]);
        lp += log_beta_pdf(w, 5.0, 5.0) + log(w) + log1p(-w);
      }
      for (int j = 0; j <= q; ++j) lp += normal_logpdf(th[p + j], 0.0, 1.0);
      lp += log_half_normal(sigma, 1.0) + th[p + q + 1];
      return lp;
    }
    case PCVG_FAMILY_RAT_GROWTH: { /* rat_growth.cpp:65-109 */
      const int base = rat_mu_a(m);
      const double mu_a = th[base];
      if (m->per_subject) {
        const double mu_b = th[base + 1];
        const double s_a = exp(th[base + 2]), s_b = exp(th[base + 3]), s_y = exp(th[base + 4]);
        const double vy = s_y * s_y;
        for (int64_t i = 0; i < m->n; ++i) {
          const double mask = excluded(m, i, fold) ? 0.0 : 1.0;
          lp += mask * normal_logpdf(m->y[i], rat_mean(m, th, i), vy);
        }
        for (int g = 0; g < J; ++g) {
          lp += normal_logpdf(th[g], mu_a, s_a * s_a);
          lp += normal_logpdf(th[J + g], mu_b, s_b * s_b);
        }
        lp += normal_logpdf(mu_a, 250.0, 20.0) + normal_logpdf(mu_b, 6.0, 2.0);
        lp += log_gamma_pdf(s_a, 25.0, 2.0) + th[base + 2];
        lp += log_gamma_pdf(s_b, 5.0, 10.0) + th[base + 3];
        lp += log_gamma_pdf(s_y, 1.0, 2.0) + th[base + 4];
      } else {
        const double s_a = exp(th[base + 1]), s_y = exp(th[base + 2]);
        const double vy = s_y * s_y;
        for (int64_t i = 0; i < m->n; ++i) {
          const double mask = excluded(m, i, fold) ? 0.0 : 1.0;
          lp += mask * normal_logpdf(m->y[i], rat_mean(m, th, i), vy);
        }
        for (int g = 0; g < J; ++g) lp += normal_logpdf(th[g], mu_a, s_a * s_a);
        lp += normal_logpdf(th[J], 6.0, 2.0);
        lp += normal_logpdf(mu_a, 250.0, 20.0);
        lp += log_gamma_pdf(s_a, 25.0, 2.0) + th[base + 1];
        lp += log_gamma_pdf(s_y, 1.0, 2.0) + th[base + 2];
      }
      return lp;
    }
    case PCVG_FAMILY_LOGISTIC: { /* oracle/ref_plugins.cpp LogisticModel::log_joint */
      for (int64_t i = 0; i < m->n; ++i) {
        const double mask = excluded(m, i, fold) ? 0.0 : 1.0;
        const double t = logit_eta(m, th, i);
        lp += mask * (m->y[i] * t - softplus(t));
      }
      for (int j = 0; j <= m->P; ++j) lp += normal_logpdf(th[j], 0.0, 1.0);
      return lp;
    }
  }
  return NAN;
}

/* Delegating fault injection of the reference's engine test (BrokenFoldModel, test_engine.cpp:57-90):
 * every gradient on `fold` is NaN, so that fold's chains diverge on every step. */
void pcvo_model_break_fold(pcvo_model* m, int32_t fold) { m->broken_fold = fold; }

static void grad_impl(const pcvo_model* m, const double* th, int32_t fold, double* grad);
void pcvo_grad(const pcvo_model* m, const double* th, int32_t fold, double* grad) {
  grad_impl(m, th, fold, grad);
  if (fold == m->broken_fold)
    for (int i = 0; i < m->dim; ++i) grad[i] = NAN;
}

static void grad_impl(const pcvo_model* m, const double* th, int32_t fold, double* grad) {
  const int J = m->J;
  for (int i = 0; i < m->dim; ++i) grad[i] = 0.0;
  switch (m->family) {
    case PCVG_FAMILY_GROUPED: { /* grouped_regression.cpp:87-122 */
      const int P = m->P;
      const double* beta = th + J;
      const double mu_a = th[J + P];
      const double sig_a = exp(th[J + P + 1]);
      const double sig_y = exp(th[J + P + 2]);
      const double va = sig_a * sig_a, vy = sig_y * sig_y;
      double sum_r2 = 0.0;
      long n_train = 0;
      for (int64_t i = 0; i < m->n; ++i) {
        if (excluded(m, i, fold)) continue;
        const double r = m->y[i] - grouped_linpred(m, th, i);
        grad[m->g[i]] += r / vy;
        for (int p = 0; p < P; ++p)
          if (m->mask[p]) grad[J + p] += xv(m, i, p) * r / vy;
        sum_r2 += r * r;
        ++n_train;
      }
      double sum_a2 = 0.0;
      for (int g = 0; g < J; ++g) {
        const double dev = th[g] - mu_a;
        grad[g] -= dev / va;
        grad[J + P] += dev / va;
        sum_a2 += dev * dev;
      }
      grad[J + P] -= mu_a;
      for (int p = 0; p < P; ++p) grad[J + p] -= beta[p];
      grad[J + P + 1] = sum_a2 / va - J - va / 10.0 + 1.0;
      grad[J + P + 2] = sum_r2 / vy - n_train - vy / 10.0 + 1.0;
      return;
    }
    case PCVG_FAMILY_RADON: { /* radon.cpp:76-107 */
      const double beta = th[J], mu_a = th[J + 1];
      const double va = exp(th[J + 2]), vy = exp(th[J + 3]);
      const double sa = sqrt(va);
      const double bmask = m->include_floor ? 1.0 : 0.0;
      double sum_r2 = 0.0, sum_rz = 0.0;
      long n_train = 0;
      for (int64_t i = 0; i < m->n; ++i) {
        if (excluded(m, i, fold)) continue;
        const int g = m->g[i];
        const double mean = mu_a + sa * th[g] + bmask * beta * xv(m, i, 0);
        const double r = m->y[i] - mean;
        grad[g] += sa * r / vy;
        if (m->include_floor) grad[J] += xv(m, i, 0) * r / vy;
        grad[J + 1] += r / vy;
        sum_r2 += r * r;
        sum_rz += r * th[g];
        ++n_train;
      }
      for (int g = 0; g < J; ++g) grad[g] -= th[g];
      grad[J] -= beta;
      grad[J + 1] -= mu_a / 4.0;
      grad[J + 2] = 0.5 * sa * sum_rz / vy + 6.0 - 9.0 * va;
      grad[J + 3] = 0.5 * (sum_r2 / vy - n_train) + 10.0 - 10.0 * vy;
      return;
    }
    case PCVG_FAMILY_SEASONAL_AR: { /* seasonal_ar.cpp:79-105 */
      const int p = m->p, q = m->q;
      const double sigma = exp(th[p + q + 1]);
      const double v = sigma * sigma;
      double sum_r2 = 0.0;
      long n_train = 0;
      for (int64_t i = 0; i < m->n; ++i) {
        if (excluded(m, i, fold)) continue;
        const double r = m->y[i] - seasonal_mean(m, th, i);
        for (int a = 0; a < p; ++a) grad[a] += r * xv(m, i, a) * drho_du(m, th[a]) / v;
        grad[p] += r / v;
        for (int j = 0; j < q; ++j) grad[p + 1 + j] += r * xv(m, i, p + j) / v;
        sum_r2 += r * r;
        ++n_train;
      }
      for (int a = 0; a < p; ++a) {
        const double w = logistic_fn(th[a]);
        grad[a] += 4.0 * (1.0 - w) - 4.0 * w + 1.0 - 2.0 * w;
      }
      for (int j = 0; j <= q; ++j) grad[p + j] -= th[p + j];
      grad[p + q + 1] = sum_r2 / v - n_train - v + 1.0;
      return;
    }
    case PCVG_FAMILY_RAT_GROWTH: { /* rat_growth.cpp:111-172 */
      const int base = rat_mu_a(m);
      const double mu_a = th[base];
      if (m->per_subject) {
        const double mu_b = th[base + 1];
        const double s_a = exp(th[base + 2]), s_b = exp(th[base + 3]), s_y = exp(th[base + 4]);
        const double va = s_a * s_a, vb = s_b * s_b, vy = s_y * s_y;
        double sum_r2 = 0.0;
        long n_train = 0;
        for (int64_t i = 0; i < m->n; ++i) {
          if (excluded(m, i, fold)) continue;
          const int g = m->g[i];
          const double t = xv(m, i, 0);
          const double r = m->y[i] - rat_mean(m, th, i);
          grad[g] += r / vy;
          grad[J + g] += t * r / vy;
          sum_r2 += r * r;
          ++n_train;
        }
        double sum_a2 = 0.0, sum_b2 = 0.0;
        for (int g = 0; g < J; ++g) {
          const double da = th[g] - mu_a, db = th[J + g] - mu_b;
          grad[g] -= da / va;
          grad[J + g] -= db / vb;
          grad[base] += da / va;
          grad[base + 1] += db / vb;
          sum_a2 += da * da;
          sum_b2 += db * db;
        }
        grad[base] -= (mu_a - 250.0) / 20.0;
        grad[base + 1] -= (mu_b - 6.0) / 2.0;
        grad[base + 2] = sum_a2 / va - J + 25.0 - 2.0 * s_a;
        grad[base + 3] = sum_b2 / vb - J + 5.0 - 10.0 * s_b;
        grad[base + 4] = sum_r2 / vy - n_train + 1.0 - 2.0 * s_y;
      } else {
        const double s_a = exp(th[base + 1]), s_y = exp(th[base + 2]);
        const double va = s_a * s_a, vy = s_y * s_y;
        double sum_r2 = 0.0;
        long n_train = 0;
        for (int64_t i = 0; i < m->n; ++i) {
          if (excluded(m, i, fold)) continue;
          const int g = m->g[i];
          const double t = xv(m, i, 0);
          const double r = m->y[i] - rat_mean(m, th, i);
          grad[g] += r / vy;
          grad[J] += t * r / vy;
          sum_r2 += r * r;
          ++n_train;
        }
        double sum_a2 = 0.0;
        for (int g = 0; g < J; ++g) {
          const double da = th[g] - mu_a;
          grad[g] -= da / va;
          grad[base] += da / va;
          sum_a2 += da * da;
        }
        grad[J] -= (th[J] - 6.0) / 2.0;
        grad[base] -= (mu_a - 250.0) / 20.0;
        grad[base + 1] = sum_a2 / va - J + 25.0 - 2.0 * s_a;
        grad[base + 2] = sum_r2 / vy - n_train + 1.0 - 2.0 * s_y;
      }
      return;
    }
    case PCVG_FAMILY_LOGISTIC: { /* oracle/ref_plugins.cpp LogisticModel::grad_log_joint */
      for (int64_t i = 0; i < m->n; ++i) {
        if (excluded(m, i, fold)) continue;
        const double r = m->y[i] - sigmoid(logit_eta(m, th, i));
        grad[0] += r;
        for (int p = 0; p < m->P; ++p) grad[1 + p] += xv(m, i, p) * r;
      }
      for (int j = 0; j <= m->P; ++j) grad[j] -= th[j];
      return;
    }
  }
}

double pcvo_log_pred(const pcvo_model* m, const double* th, int32_t fold) {
  if (fold >= m->K) return 0.0;
  const int J = m->J;
  double lp = 0.0;
  double yv[4096], mv[4096];
  for (int64_t s = m->fold_seg[fold]; s < m->fold_seg[fold + 1]; ++s) {
    const int64_t r0 = m->seg_row[s], r1 = m->seg_row[s + 1];
    switch (m->family) {
      case PCVG_FAMILY_GROUPED: { /* grouped_regression.cpp:124-163 */
        const int P = m->P;
        const double mu_a = th[J + P];
        const double sig_a = exp(th[J + P + 1]);
        const double sig_y = exp(th[J + P + 2]);
        const double va = sig_a * sig_a, vy = sig_y * sig_y;
        if (m->seg_unseen[s]) {
          int nn = 0;
          for (int64_t t = r0; t < r1 && nn < 4096; ++t, ++nn) {
            const int64_t i = m->rows[t];
            yv[nn] = m->y[i];
            double mm = 0.0;
            for (int p = 0; p < P; ++p)
              if (m->mask[p]) mm += xv(m, i, p) * th[J + p];
            mv[nn] = mu_a + mm;
          }
          if (!(vy > 0.0) || va < 0.0) return NAN; /* numeric_fault (grouped_regression.cpp:128-129) */
          lp += mvn_logpdf_compound(yv, mv, nn, vy, va);
        } else {
          for (int64_t t = r0; t < r1; ++t)
            lp += normal_logpdf(m->y[m->rows[t]], grouped_linpred(m, th, m->rows[t]), vy);
        }
        break;
      }
      case PCVG_FAMILY_RADON: { /* radon.cpp:109-138 */
        const double beta = th[J], mu_a = th[J + 1];
        const double va = exp(th[J + 2]), vy = exp(th[J + 3]);
        const double bmask = m->include_floor ? 1.0 : 0.0;
        if (m->seg_unseen[s]) {
          int nn = 0;
          for (int64_t t = r0; t < r1 && nn < 4096; ++t, ++nn) {
            const int64_t i = m->rows[t];
            yv[nn] = m->y[i];
            mv[nn] = mu_a + bmask * beta * xv(m, i, 0);
          }
          lp += mvn_logpdf_compound(yv, mv, nn, vy, va);
        } else {
          for (int64_t t = r0; t < r1; ++t) {
            const int64_t i = m->rows[t];
            const double mean = mu_a + sqrt(va) * th[m->seg_group[s]] + bmask * beta * xv(m, i, 0);
            lp += normal_logpdf(m->y[i], mean, vy);
          }
        }
        break;
      }
      case PCVG_FAMILY_SEASONAL_AR: { /* seasonal_ar.cpp:107-115 */
        const double v = exp(2.0 * th[m->p + m->q + 1]);
        for (int64_t t = r0; t < r1; ++t)
          lp += normal_logpdf(m->y[m->rows[t]], seasonal_mean(m, th, m->rows[t]), v);
        break;
      }
      case PCVG_FAMILY_LOGISTIC:
        for (int64_t t = r0; t < r1; ++t) {
          const int64_t i = m->rows[t];
          const double e = logit_eta(m, th, i);
          lp += m->y[i] * e - softplus(e);
        }
        break;
      case PCVG_FAMILY_RAT_GROWTH: { /* rat_growth.cpp:174-226 */
        const int base = rat_mu_a(m);
        const double mu_a = th[base];
        if (m->per_subject) {
          const double mu_b = th[base + 1];
          const double va = exp(2.0 * th[base + 2]), vb = exp(2.0 * th[base + 3]);
          const double vy = exp(2.0 * th[base + 4]);
          if (m->seg_unseen[s]) {
            const int nn = (int)(r1 - r0);
            if (nn > 64) return NAN;
            double cov[64 * 64];
            for (int a = 0; a < nn; ++a) {
              const double ta = xv(m, m->rows[r0 + a], 0);
              yv[a] = m->y[m->rows[r0 + a]];
              mv[a] = mu_a + mu_b * ta;
              for (int b = 0; b < nn; ++b) {
                const double tb = xv(m, m->rows[r0 + b], 0);
                cov[a * nn + b] = va + vb * ta * tb + (a == b ? vy : 0.0);
              }
            }
            lp += mvn_logpdf_chol(yv, mv, cov, nn);
          } else {
            for (int64_t t = r0; t < r1; ++t)
              lp += normal_logpdf(m->y[m->rows[t]], rat_mean(m, th, m->rows[t]), vy);
          }
        } else {
          const double va = exp(2.0 * th[base + 1]), vy = exp(2.0 * th[base + 2]);
          const double beta = th[J];
          if (m->seg_unseen[s]) {
            int nn = 0;
            for (int64_t t = r0; t < r1 && nn < 4096; ++t, ++nn) {
              const int64_t i = m->rows[t];
              yv[nn] = m->y[i];
              mv[nn] = mu_a + beta * xv(m, i, 0);
            }
            lp += mvn_logpdf_compound(yv, mv, nn, vy, va);
          } else {
            for (int64_t t = r0; t < r1; ++t)
              lp += normal_logpdf(m->y[m->rows[t]], rat_mean(m, th, m->rows[t]), vy);
          }
        }
        break;
      }
    }
  }
  return lp;
}

/* Model::pred_derivs / pred_sample over the fold's test rows in fold_meta order:
 * grouped_regression.cpp:190-213, radon.cpp:167-199, seasonal_ar.cpp:133-150. The logistic
 * family (binary outcome) supports neither (Model defaults, model.hpp:54-66). */
static int64_t test_row(const pcvo_model* m, int32_t fold, int64_t t) {
  return m->rows[m->seg_row[m->fold_seg[fold]] + t];
}
static int pred_mean_scale(const pcvo_model* m, const double* th, int32_t fold, int64_t t,
                           double* mean, double* var, double* sd) {
  const int64_t i = test_row(m, fold, t);
  const int J = m->J;
  switch (m->family) {
    case PCVG_FAMILY_GROUPED: {
      const double sig_y = exp(th[J + m->P + 2]);
      *var = sig_y * sig_y;
      *sd = sig_y;
      *mean = grouped_linpred(m, th, i);
      return 1;
    }
    case PCVG_FAMILY_RADON: {
      /* locate the test row's county: the segment holding t */
      int64_t s = m->fold_seg[fold];
      const int64_t pos = m->seg_row[m->fold_seg[fold]] + t;
      while (m->seg_row[s + 1] <= pos) ++s;
      const double beta = th[J], mu_a = th[J + 1];
      const double sa = exp(0.5 * th[J + 2]);
      const double bmask = m->include_floor ? 1.0 : 0.0;
      *var = exp(th[J + 3]);
      *sd = exp(0.5 * th[J + 3]);
      *mean = mu_a + sa * th[m->seg_group[s]] + bmask * beta * xv(m, i, 0);
      return 1;
    }
    case PCVG_FAMILY_SEASONAL_AR:
      *var = exp(2.0 * th[m->p + m->q + 1]);
      *sd = exp(th[m->p + m->q + 1]);
      *mean = seasonal_mean(m, th, i);
      return 1;
    case PCVG_FAMILY_RAT_GROWTH: { /* rat_growth.cpp:267-290 */
      const double s_y = exp(th[m->dim - 1]);
      *var = s_y * s_y;
      *sd = s_y;
      *mean = rat_mean(m, th, i);
      return 1;
    }
  }
  return 0;
}
int pcvo_supports_pred(const pcvo_model* m) { return m->family != PCVG_FAMILY_LOGISTIC; }
void pcvo_pred_derivs(const pcvo_model* m, const double* th, int32_t fold, double* d1, double* d2) {
  const int64_t n = pcvo_test_size(m, fold);
  for (int64_t t = 0; t < n; ++t) {
    double mean, var, sd;
    pred_mean_scale(m, th, fold, t, &mean, &var, &sd);
    d1[t] = -(m->y[test_row(m, fold, t)] - mean) / var;
    d2[t] = -1.0 / var;
  }
}
void pcvo_pred_sample(const pcvo_model* m, const double* th, int32_t fold, pcvo_rng* rng, double* out) {
  const int64_t n = pcvo_test_size(m, fold);
  for (int64_t t = 0; t < n; ++t) {
    double mean, var, sd;
    pred_mean_scale(m, th, fold, t, &mean, &var, &sd);
    out[t] = mean + sd * pcvo_normal(rng);
  }
}

int pcvo_pred_sample_stream(const pcvo_model* m, const double* theta, int32_t fold, uint64_t seed,
                            uint64_t stream, int32_t times, double* out) {
  if (!pcvo_supports_pred(m)) return PCVG_UNSUPPORTED_SCORE;
  pcvo_rng rng;
  pcvo_rng_init(&rng, seed, stream);
  const int64_t n = pcvo_test_size(m, fold);
  for (int32_t r = 0; r < times; ++r) pcvo_pred_sample(m, theta, fold, &rng, out + r * n);
  return 0;
}

/* ------------------------------------------------------------------ hmc.cpp:22-99 */
static int all_finite(const double* v, int n) {
  for (int i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

int32_t pcvo_leapfrog(const pcvo_model* m, int32_t fold, double step, int32_t n_lf,
                      const double* inv_mass, double* q, double* p) { /* hmc.cpp:22-51 */
  const int d = m->dim;
  double* q0 = malloc(sizeof(double) * d);
  double* p0 = malloc(sizeof(double) * d);
  double* grad = malloc(sizeof(double) * d);
  memcpy(q0, q, sizeof(double) * d);
  memcpy(p0, p, sizeof(double) * d);
  int ok = 1;
  pcvo_grad(m, q, fold, grad);
  if (!all_finite(grad, d)) { ok = 0; goto done; }
  const double half = 0.5 * step;
  for (int i = 0; i < d; ++i) p[i] += half * grad[i];
  for (int s = 0; s < n_lf; ++s) {
    for (int i = 0; i < d; ++i) q[i] += step * inv_mass[i] * p[i];
    if (!all_finite(q, d)) { ok = 0; goto done; }
    pcvo_grad(m, q, fold, grad);
    if (!all_finite(grad, d)) { ok = 0; goto done; }
    const double scale = (s == n_lf - 1) ? half : step;
    for (int i = 0; i < d; ++i) p[i] += scale * grad[i];
    if (!all_finite(p, d)) { ok = 0; goto done; }
  }
done:
  if (!ok) {
    memcpy(q, q0, sizeof(double) * d);
    memcpy(p, p0, sizeof(double) * d);
  }
  free(q0); free(p0); free(grad);
  return ok;
}

static double kinetic(const double* inv_mass, const double* p, int d) {
  double k = 0.0;
  for (int i = 0; i < d; ++i) k += inv_mass[i] * p[i] * p[i];
  return 0.5 * k;
}

/* hmc.cpp:53-99; `draw_u` supplies the Metropolis uniform (the chain RNG or an injection).
 * Returns divergent flag; *accepted set. */
typedef double (*u_source)(void*);
static int hmc_core(const pcvo_model* m, int32_t fold, double step, int32_t n_lf,
                    const double* inv_mass, double* position, const double* momentum,
                    u_source draw_u, void* u_ctx, double* h0_out, double* h1_out,
                    int32_t* accepted, double* wq, double* wp) {
  const int d = m->dim;
  const double h0 = -pcvo_log_joint(m, position, fold) + kinetic(inv_mass, momentum, d);
  memcpy(wq, position, sizeof(double) * d);
  memcpy(wp, momentum, sizeof(double) * d);
  const int ok = pcvo_leapfrog(m, fold, step, n_lf, inv_mass, wq, wp);
  const double h1 = ok ? -pcvo_log_joint(m, wq, fold) + kinetic(inv_mass, wp, d) : NAN;
  const double dh = h1 - h0;
  if (h0_out) *h0_out = h0;
  if (h1_out) *h1_out = h1;
  *accepted = 0;
  const int divergent = !ok || isnan(dh) || (isfinite(dh) && fabs(dh) > 1000.0);
  if (divergent) return 1;
  const double u = draw_u(u_ctx);
  if (log(u) < -dh) {
    *accepted = 1;
    memcpy(position, wq, sizeof(double) * d);
  }
  return 0;
}
static double u_from_rng(void* r) { return pcvo_uniform((pcvo_rng*)r); }
static double u_from_value(void* v) { return *(const double*)v; }

void pcvo_hmc_probe(const pcvo_model* m, int32_t fold, double step, int32_t n_lf,
                    const double* inv_mass, const double* theta, const double* momentum,
                    double u, double* theta_out, double* h0, double* h1, int32_t* accepted,
                    int32_t* divergent) {
  const int d = m->dim;
  double* wq = malloc(sizeof(double) * d);
  double* wp = malloc(sizeof(double) * d);
  memcpy(theta_out, theta, sizeof(double) * d);
  *divergent = hmc_core(m, fold, step, n_lf, inv_mass, theta_out, momentum, u_from_value, &u,
                        h0, h1, accepted, wq, wp);
  free(wq);
  free(wp);
}

/* One reference hmc_step on a chain stream (hmc.cpp:53-99, momentum rng.normal()/sqrt(m)). */
static int hmc_step_rng(const pcvo_model* m, int32_t fold, double step, int32_t n_lf,
                        const double* inv_mass, double* position, pcvo_rng* rng, double* mom,
                        double* wq, double* wp, int32_t* accepted) {
  const int d = m->dim;
  for (int i = 0; i < d; ++i) mom[i] = pcvo_normal(rng) / sqrt(inv_mass[i]);
  return hmc_core(m, fold, step, n_lf, inv_mass, position, mom, u_from_rng, rng, NULL, NULL,
                  accepted, wq, wp);
}

int pcvo_hmc_chain(const pcvo_model* m, int32_t fold, double step, int32_t n_lf,
                   const double* inv_mass, uint64_t seed, uint64_t stream, const double* theta0,
                   int64_t n_steps, double* traj, int32_t* divergent) {
  const int d = m->dim;
  pcvo_rng rng;
  pcvo_rng_init(&rng, seed, stream);
  double* pos = malloc(sizeof(double) * d);
  double* mom = malloc(sizeof(double) * d);
  double* wq = malloc(sizeof(double) * d);
  double* wp = malloc(sizeof(double) * d);
  memcpy(pos, theta0, sizeof(double) * d);
  for (int64_t s = 0; s < n_steps; ++s) {
    int32_t acc;
    const int div = hmc_step_rng(m, fold, step, n_lf, inv_mass, pos, &rng, mom, wq, wp, &acc);
    memcpy(traj + s * d, pos, sizeof(double) * d);
    if (divergent) divergent[s] = div;
  }
  free(pos); free(mom); free(wq); free(wp);
  return 0;
}

/* ------------------------------------------------------------------ accum.cpp:101-182 */
typedef struct {
  double u_x, u_x2;  /* LogSpaceAccumulator */
  long raw_count;
  int b;             /* BatchState */
  double z_x, v_x, v_x2;
  long committed;
  int pending;
  int D;             /* ShuffleBlocks */
  long planned_n;
  double y_x[16], y_x2[16];
  double c;
  long count, faults;
} score_accum;

static void accum_init(score_accum* a, int b, int D, long n, double c) {
  memset(a, 0, sizeof *a);
  a->u_x = a->u_x2 = NEG_INF;
  a->b = b;
  a->z_x = a->v_x = a->v_x2 = NEG_INF;
  a->D = D;
  a->planned_n = n;
  a->c = c;
}
static int block_for(long iter, long planned_n, int d) { /* accum.cpp:134-139 */
  if (planned_n <= 0) return 0;
  long blk = iter * d / planned_n;
  if (blk >= d) blk = d - 1;
  return (int)blk;
}
static void batch_add(score_accum* a, double s) { /* accum.cpp:115-127 */
  a->z_x = logaddexp(a->z_x, s);
  if (++a->pending == a->b) {
    const double log_mean = a->z_x - log((double)a->b);
    a->v_x = logaddexp(a->v_x, log_mean);
    a->v_x2 = logaddexp(a->v_x2, 2.0 * log_mean);
    a->z_x = NEG_INF;
    a->pending = 0;
    ++a->committed;
  }
}
static void accum_observe(score_accum* a, double s, long iter) { /* accum.cpp:164-182 */
  const int blk = block_for(iter, a->planned_n, a->D);
  if (isnan(s) || (isinf(s) && s > 0.0)) {
    ++a->faults;
    s = NEG_INF;
    a->u_x = logaddexp(a->u_x, s);
    a->u_x2 = logaddexp(a->u_x2, 2.0 * s);
    ++a->raw_count;
    batch_add(a, s);
    a->y_x[blk] += 0.0;
    a->y_x2[blk] += 0.0 * 0.0;
    ++a->count;
    return;
  }
  a->u_x = logaddexp(a->u_x, s);
  a->u_x2 = logaddexp(a->u_x2, 2.0 * s);
  ++a->raw_count;
  batch_add(a, s);
  a->y_x[blk] += s - a->c;
  a->y_x2[blk] += (s - a->c) * (s - a->c);
  ++a->count;
}

/* ------------------------------------------------------------------ scoring / diagnostics */
typedef struct {
  double estimate, log_f_hat, mc, naive, ess;
  long batches;
  int fault;
} fold_score;

static fold_score logs_fold_score(const score_accum* const* ch, int l, long n) { /* scoring.cpp:10-62 */
  fold_score fs;
  memset(&fs, 0, sizeof fs);
  const double ln = (double)l * (double)n;
  double ux[256];
  for (int c = 0; c < l; ++c) {
    ux[c] = ch[c]->u_x;
    fs.fault = fs.fault || ch[c]->faults > 0;
    fs.batches += ch[c]->committed;
  }
  const double lf = logsumexp(ux, l) - log(ln);
  fs.estimate = lf;
  fs.log_f_hat = lf;
  if (lf == NEG_INF) {
    fs.fault = 1;
    fs.mc = INFINITY;
    fs.naive = INFINITY;
    fs.ess = NAN;
    return fs;
  }
  double sum_u2 = 0.0;
  for (int c = 0; c < l; ++c) sum_u2 += exp(ch[c]->u_x2 - 2.0 * lf);
  fs.naive = ln > 1 ? (sum_u2 - ln) / (ln - 1.0) : 0.0;
  if (fs.naive < 0.0) fs.naive = 0.0;
  const long a = ch[0]->committed;
  const long la = fs.batches;
  const int b = ch[0]->b;
  if (la >= 2 && a >= 1) {
    double ss = 0.0;
    for (int c = 0; c < l; ++c) {
      const double s2 = exp(ch[c]->v_x2 - 2.0 * lf);
      const double s1 = exp(ch[c]->v_x - lf);
      ss += s2 - 2.0 * s1 + (double)ch[c]->committed;
    }
    fs.mc = b * ss / (la - 1.0);
    if (fs.mc < 0.0) fs.mc = 0.0;
    fs.ess = fs.mc > 0.0 ? ln * fs.naive / fs.mc : NAN;
  } else {
    fs.mc = NAN;
    fs.ess = NAN;
  }
  return fs;
}

int pcvo_rhat_from_sums(const double* sx, const double* sxx, int32_t l, int64_t n, double* w_out,
                        double* b_out, double* rhat) { /* diagnostics.cpp:11-33 */
  if (l < 2 || n < 2) return 0;
  double w = 0.0, grand = 0.0;
  for (int c = 0; c < l; ++c) {
    w += (sxx[c] - sx[c] * sx[c] / n) / (n - 1.0) / l;
    grand += sx[c] / n / l;
  }
  double b = 0.0;
  for (int c = 0; c < l; ++c) {
    const double dev = sx[c] / n - grand;
    b += dev * dev;
  }
  b *= (double)n / (l - 1.0);
  if (!isfinite(w) || !isfinite(b) || !(w > 0.0)) return 0;
  if (w_out) *w_out = w;
  if (b_out) *b_out = b;
  *rhat = sqrt(((n - 1.0) / n * w + b / n) / w);
  return 1;
}

static int rhat_from_blocks(const score_accum* const* ch, int l, long n, double* rhat) { /* diagnostics.cpp:35-44 */
  double sx[256], sxx[256];
  for (int c = 0; c < l; ++c) {
    double s = 0.0, s2 = 0.0;
    for (int d = 0; d < ch[c]->D; ++d) s += ch[c]->y_x[d];
    for (int d = 0; d < ch[c]->D; ++d) s2 += ch[c]->y_x2[d];
    sx[c] = s;
    sxx[c] = s2;
  }
  return pcvo_rhat_from_sums(sx, sxx, l, n, NULL, NULL, rhat);
}

double pcvo_selection_probability(double delta_hat, const double* deltas, int64_t k,
                                  double* sigma2) { /* scoring.cpp:141-158 */
  const double mean = delta_hat / k;
  double ss = 0.0;
  for (int64_t i = 0; i < k; ++i) ss += (deltas[i] - mean) * (deltas[i] - mean);
  *sigma2 = ss / (k - 1.0);
  const double denom = sqrt(k * *sigma2);
  if (denom == 0.0) return delta_hat > 0.0 ? 1.0 : (delta_hat < 0.0 ? 0.0 : 0.5);
  return normal_cdf(delta_hat / denom);
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}
double pcvo_benchmark_quantile(const double* values, int64_t n, double q) { /* diagnostics.cpp:103-119 */
  double* s = malloc(sizeof(double) * n);
  memcpy(s, values, sizeof(double) * n);
  qsort(s, n, sizeof(double), cmp_double);
  long rank = (long)ceil(q * n);
  if (rank < 1) rank = 1;
  if (rank > n) rank = n;
  const double v = s[rank - 1];
  free(s);
  return v;
}

/* ------------------------------------------------------------------ engine.cpp:257-483 */
typedef struct {
  int model, fold, chain;
  double* position;
  pcvo_rng rng;
  long divergences;
  double warm_logpred;
  long sampling_divergences;
  score_accum acc;
  score_accum* snaps;
  /* HS / DSS (engine.cpp:322-373): WelfordDiag of xi (2m) or WelfordAccumulator of draws (m);
   * warm-up sums (WarmupStats hs1/hs2/pred). x_acc = [a_x | a_x2] (HS) or [a_x | a_xx m*m] (DSS). */
  int64_t msize;
  double* x_warm;
  double* x_acc;
  double** x_snaps;
} chain_task;

typedef struct {
  int32_t n_models;
  pcvo_model** models;
  const int32_t* model_ids;
  const pcvg_kernel* kernels;
  const double* const* banks;
  const int64_t* bank_rows;
  const pcvg_run_config* cfg;
  chain_task* tasks;
  long n_tasks;
  double** centers; /* [m][k] */
  double*** x_centers; /* [m][k] -> hs_c (2m) / pred_c (m) */
  int b;
  long* checkpoints;
  int n_ckpt;
  int phase;
  atomic_long next;
} run_ctx;

static void task_step2(run_ctx* rc, chain_task* t) { /* engine.cpp:296-313 */
  const pcvg_run_config* cfg = rc->cfg;
  const pcvo_model* m = rc->models[t->model];
  const int d = m->dim;
  const uint64_t sm = cfg->shared_streams ? 0u : (uint64_t)rc->model_ids[t->model];
  pcvo_rng init;
  pcvo_rng_init(&init, cfg->seed, pcvo_stream_key(PCVG_STREAM_CHAIN_INIT, sm, (uint64_t)t->fold, (uint64_t)t->chain));
  const uint64_t row = pcvo_below(&init, (uint64_t)rc->bank_rows[t->model]);
  memcpy(t->position, rc->banks[t->model] + row * d, sizeof(double) * d);
  pcvo_rng_init(&t->rng, cfg->seed, pcvo_stream_key(PCVG_STREAM_CHAIN_SAMPLING, sm, (uint64_t)t->fold, (uint64_t)t->chain));
  double* mom = malloc(sizeof(double) * d);
  double* wq = malloc(sizeof(double) * d);
  double* wp = malloc(sizeof(double) * d);
  const pcvg_kernel* kp = &rc->kernels[t->model];
  t->warm_logpred = 0.0; /* warmup_discard, hmc.cpp:121-149 */
  const int64_t ms = t->msize;
  double* d1 = malloc(sizeof(double) * (ms + 1));
  double* d2 = malloc(sizeof(double) * (ms + 1));
  for (long i = 0; i < cfg->warmup; ++i) {
    int32_t acc;
    t->divergences += hmc_step_rng(m, t->fold, kp->step_size, kp->n_leapfrog, kp->inv_mass_diag,
                                   t->position, &t->rng, mom, wq, wp, &acc);
    t->warm_logpred += pcvo_log_pred(m, t->position, t->fold);
    if (cfg->score == PCVG_SCORE_HS) {
      pcvo_pred_derivs(m, t->position, t->fold, d1, d2);
      for (int64_t o = 0; o < ms; ++o) {
        t->x_warm[o] += d2[o] + d1[o] * d1[o];
        t->x_warm[ms + o] += d1[o];
      }
    } else if (cfg->score == PCVG_SCORE_DSS) {
      pcvo_pred_sample(m, t->position, t->fold, &t->rng, d1);
      for (int64_t o = 0; o < ms; ++o) t->x_warm[o] += d1[o];
    }
  }
  free(d1); free(d2);
  free(mom); free(wq); free(wp);
}

static void task_step3(run_ctx* rc, chain_task* t) { /* engine.cpp:342-381 */
  const pcvg_run_config* cfg = rc->cfg;
  const pcvo_model* m = rc->models[t->model];
  const int d = m->dim;
  const pcvg_kernel* kp = &rc->kernels[t->model];
  accum_init(&t->acc, rc->b, cfg->blocks, cfg->iters, rc->centers[t->model][t->fold]);
  double* mom = malloc(sizeof(double) * d);
  double* wq = malloc(sizeof(double) * d);
  double* wp = malloc(sizeof(double) * d);
  const long before = t->divergences;
  int next_ck = 0;
  const int64_t ms = t->msize;
  const double* xc = cfg->score != PCVG_SCORE_LOGS ? rc->x_centers[t->model][t->fold] : NULL;
  double* d1 = malloc(sizeof(double) * (2 * ms + 1));
  double* d2 = malloc(sizeof(double) * (ms + 1));
  const int64_t xlen = cfg->score == PCVG_SCORE_HS ? 4 * ms : (cfg->score == PCVG_SCORE_DSS ? ms + ms * ms : 0);
  for (long iter = 0; iter < cfg->iters; ++iter) {
    int32_t acc;
    t->divergences += hmc_step_rng(m, t->fold, kp->step_size, kp->n_leapfrog, kp->inv_mass_diag,
                                   t->position, &t->rng, mom, wq, wp, &acc);
    const double s = pcvo_log_pred(m, t->position, t->fold);
    accum_observe(&t->acc, s, iter);
    if (cfg->score == PCVG_SCORE_HS) { /* WelfordDiag::add, accum.cpp:66-74 */
      pcvo_pred_derivs(m, t->position, t->fold, d1, d2);
      for (int64_t o = 0; o < ms; ++o) {
        const double x1 = d2[o] + d1[o] * d1[o], x2 = d1[o];
        const double a = x1 - xc[o], b = x2 - xc[ms + o];
        t->x_acc[o] += a;
        t->x_acc[2 * ms + o] += a * a;
        t->x_acc[ms + o] += b;
        t->x_acc[3 * ms + o] += b * b;
      }
    } else if (cfg->score == PCVG_SCORE_DSS) { /* WelfordAccumulator::add, accum.cpp:19-26 */
      pcvo_pred_sample(m, t->position, t->fold, &t->rng, d1);
      double* axx = t->x_acc + ms;
      for (int64_t i = 0; i < ms; ++i) {
        const double di = d1[i] - xc[i];
        t->x_acc[i] += di;
        for (int64_t j = 0; j <= i; ++j) axx[i * ms + j] += di * (d1[j] - xc[j]);
      }
    }
    if (next_ck < rc->n_ckpt && iter + 1 == rc->checkpoints[next_ck]) {
      if (xlen) memcpy(t->x_snaps[next_ck], t->x_acc, sizeof(double) * xlen);
      t->snaps[next_ck++] = t->acc;
    }
  }
  t->sampling_divergences = t->divergences - before;
  free(d1); free(d2);
  free(mom); free(wq); free(wp);
}

static void* worker(void* arg) {
  run_ctx* rc = arg;
  for (;;) {
    const long i = atomic_fetch_add(&rc->next, 1);
    if (i >= rc->n_tasks) return NULL;
    if (rc->phase == 2) task_step2(rc, &rc->tasks[i]);
    else task_step3(rc, &rc->tasks[i]);
  }
}

static void run_phase(run_ctx* rc, int phase, int threads) { /* parallel_for, engine.cpp:32-61 */
  rc->phase = phase;
  atomic_store(&rc->next, 0);
  if (threads <= 1) {
    worker(rc);
    return;
  }
  pthread_t* th = malloc(sizeof(pthread_t) * threads);
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, worker, rc);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  free(th);
}

typedef struct {
  double delta_hat, mcse, sigma2, epistemic_se, prob, ess, rhat_max;
} ckpt_stats;

/* Cholesky pieces, math.hpp:46-76 (row-major, lower factor in place). */
static int cholesky_in_place(double* a, int n) {
  for (int j = 0; j < n; ++j) {
    double d = a[j * n + j];
    for (int k = 0; k < j; ++k) d -= a[j * n + k] * a[j * n + k];
    if (!(d > 0.0) || !isfinite(d)) return 0;
    const double l = sqrt(d);
    a[j * n + j] = l;
    for (int i = j + 1; i < n; ++i) {
      double s = a[i * n + j];
      for (int k = 0; k < j; ++k) s -= a[i * n + k] * a[j * n + k];
      a[i * n + j] = s / l;
    }
  }
  return 1;
}

/* Chain-merged HS / DSS estimate of one fold (engine.cpp:148-171): WelfordDiag/WelfordAccumulator
 * ::merge in chain order (accum.cpp:28-34, 76-84), hs_fold_score negated (scoring.cpp:64-73),
 * dss_fold_score (scoring.cpp:75-104). Returns 0 where the reference throws (NaN + fault). */
static int extra_fold_estimate(const pcvg_run_config* cfg, const pcvo_model* mdl, int fold,
                               const double* const* acc, int l, long count_total, int64_t ms,
                               const double* xc, double* est, int* ridged) {
  *ridged = 0;
  if (cfg->score == PCVG_SCORE_HS) {
    double score = 0.0;
    for (int64_t i = 0; i < ms; ++i) {
      double a1 = acc[0][i], a2 = acc[0][ms + i];
      for (int c = 1; c < l; ++c) { a1 += acc[c][i]; a2 += acc[c][ms + i]; }
      const double mu1 = a1 / count_total + xc[i];
      const double mu2 = a2 / count_total + xc[ms + i];
      score += 2.0 * mu1 - mu2 * mu2;
    }
    *est = -score;
    return 1;
  }
  const int d = (int)ms;
  if (count_total < d + 1 || count_total < 2) return 0;
  double* ax = malloc(sizeof(double) * d);
  double* axx = malloc(sizeof(double) * d * d);
  double* cov = malloc(sizeof(double) * d * d);
  double* fac = malloc(sizeof(double) * d * d);
  double* r = malloc(sizeof(double) * d);
  for (int i = 0; i < d; ++i) ax[i] = acc[0][i];
  for (int i = 0; i < d * d; ++i) axx[i] = acc[0][d + i];
  for (int c = 1; c < l; ++c) {
    for (int i = 0; i < d; ++i) ax[i] += acc[c][i];
    for (int i = 0; i < d * d; ++i) axx[i] += acc[c][d + i];
  }
  const double inv_n = 1.0 / (double)count_total, inv_nm1 = 1.0 / (double)(count_total - 1);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j <= i; ++j) {
      const double v = (axx[i * d + j] - ax[i] * ax[j] * inv_n) * inv_nm1;
      cov[i * d + j] = v;
      cov[j * d + i] = v;
    }
  memcpy(fac, cov, sizeof(double) * d * d);
  int ok = 1;
  if (!cholesky_in_place(fac, d)) {
    double tr = 0.0;
    for (int i = 0; i < d; ++i) tr += cov[i * d + i];
    const double ridge = 1e-8 * tr / d;
    for (int i = 0; i < d; ++i) cov[i * d + i] += ridge;
    memcpy(fac, cov, sizeof(double) * d * d);
    *ridged = 1;
    ok = cholesky_in_place(fac, d);
  }
  if (ok) {
    const int64_t r0 = mdl->seg_row[mdl->fold_seg[fold]];
    for (int i = 0; i < d; ++i) r[i] = mdl->y[mdl->rows[r0 + i]] - (ax[i] / count_total + xc[i]);
    for (int i = 0; i < d; ++i) {
      double sm = r[i];
      for (int k = 0; k < i; ++k) sm -= fac[i * d + k] * r[k];
      r[i] = sm / fac[i * d + i];
    }
    double quad = 0.0, ld = 0.0;
    for (int i = 0; i < d; ++i) quad += r[i] * r[i];
    for (int i = 0; i < d; ++i) ld += log(fac[i * d + i]);
    *est = -(2.0 * ld) - quad;
  }
  free(ax); free(axx); free(cov); free(fac); free(r);
  return ok;
}

/* compute_stats, engine.cpp:117-253. fs_out: [n_models*K], rhat_out same. */
static ckpt_stats compute_stats(run_ctx* rc, int K, long iter_count, int ck, const char* failed,
                                fold_score* fs_out, double* rhat_out, int* failed_out,
                                double* delta_k, int* ridged_out) {
  const int nm = rc->n_models, l = rc->cfg->chains;
  ckpt_stats out;
  const score_accum* ch[256];
  const double* xa[256];
  for (int m = 0; m < nm; ++m)
    for (int k = 0; k < K; ++k) {
      for (int c = 0; c < l; ++c) {
        const chain_task* t = &rc->tasks[((long)m * K + k) * l + c];
        ch[c] = &t->snaps[ck];
        xa[c] = t->x_snaps ? t->x_snaps[ck] : NULL;
      }
      fs_out[m * K + k] = logs_fold_score(ch, l, iter_count);
      ridged_out[m * K + k] = 0;
      if (rc->cfg->score != PCVG_SCORE_LOGS) {
        const chain_task* t0 = &rc->tasks[((long)m * K + k) * l];
        double est;
        if (extra_fold_estimate(rc->cfg, rc->models[m], k, xa, l, (long)l * iter_count, t0->msize,
                                rc->x_centers[m][k], &est, &ridged_out[m * K + k])) {
          fs_out[m * K + k].estimate = est;
        } else {
          fs_out[m * K + k].estimate = NAN;
          fs_out[m * K + k].fault = 1;
        }
      }
      double rh;
      rhat_out[m * K + k] = rhat_from_blocks(ch, l, iter_count, &rh) ? rh : NAN;
      failed_out[m * K + k] = failed && failed[k];
    }
  char* excl = calloc(K, 1);
  for (int k = 0; k < K; ++k) {
    if (failed && failed[k]) excl[k] = 1;
    if (failed)
      for (int m = 0; m < nm; ++m)
        if (isnan(fs_out[m * K + k].estimate)) excl[k] = 1;
    if (excl[k])
      for (int m = 0; m < nm; ++m) failed_out[m * K + k] = 1;
  }
  double naive_sum = 0.0, mc_sum = 0.0;
  int mc_inf = 0;
  double best = -1.0;
  for (int m = 0; m < nm; ++m)
    for (int k = 0; k < K; ++k) {
      if (excl[k]) continue;
      const fold_score* fs = &fs_out[m * K + k];
      if (isfinite(fs->mc)) {
        mc_sum += fs->mc;
        naive_sum += fs->naive;
      } else {
        mc_inf = 1;
      }
      const double r = rhat_out[m * K + k];
      if (isfinite(r) && r > best) best = r; /* rhat_max, diagnostics.cpp:46-59 */
    }
  double* inc = malloc(sizeof(double) * K);
  long ninc = 0;
  out.delta_hat = 0.0;
  for (int k = 0; k < K; ++k) {
    const double dk = nm == 2 ? fs_out[k].estimate - fs_out[K + k].estimate : fs_out[k].estimate;
    if (delta_k) delta_k[k] = dk;
    if (!excl[k]) inc[ninc++] = dk;
  }
  for (long i = 0; i < ninc; ++i) out.delta_hat += inc[i];
  if (ninc >= 2) {
    double s2;
    const double pr = pcvo_selection_probability(out.delta_hat, inc, ninc, &s2);
    out.sigma2 = s2;
    out.epistemic_se = sqrt((double)ninc * s2);
    out.prob = nm == 2 ? pr : NAN;
  } else {
    out.sigma2 = out.epistemic_se = out.prob = NAN;
  }
  const double ln = (double)l * iter_count;
  out.mcse = rc->cfg->score != PCVG_SCORE_LOGS ? NAN : (mc_inf ? INFINITY : sqrt(mc_sum / ln));
  out.ess = mc_sum > 0.0 ? (double)l * iter_count * naive_sum / mc_sum : NAN;
  out.rhat_max = best < 0.0 ? NAN : best;
  free(inc);
  free(excl);
  return out;
}

int pcvo_run_pcv(int32_t n_models, pcvo_model** models, const int32_t* model_ids,
                 const pcvg_kernel* kernels, const double* const* banks,
                 const int64_t* bank_rows, const pcvg_run_config* cfg, int32_t threads,
                 pcvg_report* rep, pcvo_task_out* tout, int32_t dim_max) {
  /* RunConfig::validate, engine.cpp:21-30; run_pcv preconditions engine.cpp:258-271 */
  const int b = cfg->batch_size > 0 ? cfg->batch_size
                                    : (int)fmax(1.0, floor(sqrt((double)cfg->iters * cfg->chains)));
  if (cfg->chains < 2) return set_err(PCVG_INVALID_INPUT, "need at least 2 chains per fold (Rhat)");
  if (cfg->iters < 1) return set_err(PCVG_INVALID_INPUT, "need at least 1 sampling iteration");
  if (cfg->warmup < 0) return set_err(PCVG_INVALID_INPUT, "warmup must be non-negative");
  if (cfg->iters < b) return set_err(PCVG_INVALID_INPUT, "chain length must cover at least one batch");
  if (cfg->blocks < 1 || cfg->blocks > 16) return set_err(PCVG_INVALID_INPUT, "oracle supports 1..16 shuffle blocks");
  if (cfg->bench_draws < 1) return set_err(PCVG_INVALID_INPUT, "need at least 1 benchmark draw");
  if (cfg->checkpoint_every < 0) return set_err(PCVG_INVALID_INPUT, "checkpoint_every must be >= 0");
  if (n_models < 1 || n_models > 2) return set_err(PCVG_INVALID_INPUT, "run_pcv takes one or two models");
  if (cfg->score < PCVG_SCORE_LOGS || cfg->score > PCVG_SCORE_DSS) return set_err(PCVG_INVALID_INPUT, "unknown score");
  for (int m = 0; m < n_models; ++m) /* Model::check_score_support, model.cpp:21-28 */
    if (cfg->score != PCVG_SCORE_LOGS && !pcvo_supports_pred(models[m]))
      return set_err(PCVG_UNSUPPORTED_SCORE, "model does not support the configured score");
  const int K = models[0]->K;
  for (int m = 0; m < n_models; ++m) {
    if (models[m]->K != K) return set_err(PCVG_INVALID_INPUT, "models must share one fold assignment");
    if (bank_rows[m] < 1) return set_err(PCVG_INVALID_INPUT, "full-data draws missing");
  }
  if (K < 2) return set_err(PCVG_INVALID_INPUT, "uncertainty estimates need at least 2 folds");
  if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  const int l = cfg->chains;
  const long n = cfg->iters;

  run_ctx rc;
  memset(&rc, 0, sizeof rc);
  rc.n_models = n_models;
  rc.models = models;
  rc.model_ids = model_ids;
  rc.kernels = kernels;
  rc.banks = banks;
  rc.bank_rows = bank_rows;
  rc.cfg = cfg;
  rc.b = b;
  long ck_cap = 2 + (cfg->checkpoint_every > 0 ? n / cfg->checkpoint_every : 0);
  rc.checkpoints = malloc(sizeof(long) * ck_cap);
  if (cfg->checkpoint_every > 0)
    for (long t = cfg->checkpoint_every; t < n; t += cfg->checkpoint_every) rc.checkpoints[rc.n_ckpt++] = t;
  rc.checkpoints[rc.n_ckpt++] = n;
  rc.n_tasks = (long)n_models * K * l;
  rc.tasks = calloc(rc.n_tasks, sizeof(chain_task));
  for (int m = 0; m < n_models; ++m)
    for (int k = 0; k < K; ++k)
      for (int c = 0; c < l; ++c) {
        chain_task* t = &rc.tasks[((long)m * K + k) * l + c];
        t->model = m;
        t->fold = k;
        t->chain = c;
        t->position = malloc(sizeof(double) * models[m]->dim);
        t->snaps = malloc(sizeof(score_accum) * rc.n_ckpt);
        t->msize = pcvo_test_size(models[m], k);
        if (cfg->score != PCVG_SCORE_LOGS) {
          const int64_t ms = t->msize;
          const int64_t xl = cfg->score == PCVG_SCORE_HS ? 4 * ms : ms + ms * ms;
          t->x_warm = calloc(2 * ms + 1, sizeof(double));
          t->x_acc = calloc(xl + 1, sizeof(double));
          t->x_snaps = malloc(sizeof(double*) * rc.n_ckpt);
          for (int ci = 0; ci < rc.n_ckpt; ++ci) t->x_snaps[ci] = calloc(xl + 1, sizeof(double));
        }
      }
  run_phase(&rc, 2, threads);
  /* centering constants, engine.cpp:316-339 */
  rc.centers = malloc(sizeof(double*) * n_models);
  for (int m = 0; m < n_models; ++m) {
    rc.centers[m] = calloc(K, sizeof(double));
    if (cfg->warmup == 0) continue;
    const double denom = (double)l * cfg->warmup;
    for (int k = 0; k < K; ++k)
      for (int c = 0; c < l; ++c) rc.centers[m][k] += rc.tasks[((long)m * K + k) * l + c].warm_logpred / denom;
  }
  /* HS / DSS centring vectors hs_c / pred_c (engine.cpp:324-338) */
  if (cfg->score != PCVG_SCORE_LOGS) {
    rc.x_centers = malloc(sizeof(double**) * n_models);
    for (int m = 0; m < n_models; ++m) {
      rc.x_centers[m] = malloc(sizeof(double*) * K);
      for (int k = 0; k < K; ++k) {
        const int64_t ms = pcvo_test_size(models[m], k);
        const int64_t wl = cfg->score == PCVG_SCORE_HS ? 2 * ms : ms;
        double* xc = calloc(wl + 1, sizeof(double));
        if (cfg->warmup > 0) {
          const double denom = (double)l * cfg->warmup;
          for (int c = 0; c < l; ++c) {
            const chain_task* t = &rc.tasks[((long)m * K + k) * l + c];
            for (int64_t e = 0; e < wl; ++e) xc[e] += t->x_warm[e] / denom;
          }
        }
        rc.x_centers[m][k] = xc;
      }
    }
  }
  run_phase(&rc, 3, threads);
  /* failed folds, engine.cpp:385-397 */
  char* failed = calloc(K, 1);
  for (int k = 0; k < K; ++k)
    for (int m = 0; m < n_models && !failed[k]; ++m) {
      int all_bad = 1;
      for (int c = 0; c < l; ++c)
        if (rc.tasks[((long)m * K + k) * l + c].sampling_divergences * 2 <= n) { all_bad = 0; break; }
      if (all_bad) failed[k] = 1;
    }
  fold_score* fs = malloc(sizeof(fold_score) * n_models * K);
  double* rh = malloc(sizeof(double) * n_models * K);
  int* fl = malloc(sizeof(int) * n_models * K);
  int* rg = malloc(sizeof(int) * n_models * K);
  rep->n_checkpoints = rc.n_ckpt;
  for (int ci = 0; ci < rc.n_ckpt; ++ci) {
    const int last = ci + 1 == rc.n_ckpt;
    const ckpt_stats st = compute_stats(&rc, K, rc.checkpoints[ci], ci, last ? failed : NULL, fs, rh, fl,
                                        last ? rep->delta_k : NULL, rg);
    double* o = rep->snapshots ? rep->snapshots + 7 * ci : NULL;
    if (o) {
      o[0] = (double)rc.checkpoints[ci];
      o[1] = st.delta_hat;
      o[2] = st.mcse;
      o[3] = st.epistemic_se;
      o[4] = st.prob;
      o[5] = st.ess;
      o[6] = st.rhat_max;
    }
    if (last) {
      rep->delta_hat = st.delta_hat;
      rep->mcse = st.mcse;
      rep->sigma2_delta = st.sigma2;
      rep->epistemic_se = st.epistemic_se;
      rep->prob_a_better = st.prob;
      rep->ess_overall = st.ess;
      rep->rhat_max = st.rhat_max;
      for (int m = 0; m < n_models; ++m) {
        rep->score_total[m] = 0.0;
        rep->numeric_faults[m] = 0;
        rep->rhat_excluded[m] = 0;
        for (int k = 0; k < K; ++k) {
          const long i = (long)m * K + k;
          rep->folds.estimate[i] = fs[i].estimate;
          rep->folds.log_f_hat[i] = fs[i].log_f_hat;
          rep->folds.mc_contribution[i] = fs[i].mc;
          if (rep->folds.naive_contribution) rep->folds.naive_contribution[i] = fs[i].naive;
          rep->folds.ess[i] = fs[i].ess;
          rep->folds.rhat[i] = rh[i];
          rep->folds.batches[i] = fs[i].batches;
          rep->folds.fault[i] = fs[i].fault;
          rep->folds.failed[i] = fl[i];
          if (rep->folds.dss_ridged) rep->folds.dss_ridged[i] = rg[i];
          for (int c = 0; c < l; ++c)
            rep->divergences[i * l + c] = rc.tasks[i * l + c].sampling_divergences;
          if (!fl[i]) rep->score_total[m] += fs[i].estimate;
          if (fs[i].fault) ++rep->numeric_faults[m];
          if (!isfinite(rh[i]) && !fl[i]) ++rep->rhat_excluded[m];
        }
      }
    }
  }
  rep->dropped_batch_draws = 0;
  for (long i = 0; i < rc.n_tasks; ++i) rep->dropped_batch_draws += rc.tasks[i].acc.pending;
  /* shuffle benchmark, engine.cpp:464-480 + diagnostics.cpp:76-101 */
  const int D = cfg->blocks;
  rep->benchmark_count = 0;
  for (int r = 0; r < cfg->bench_draws; ++r) {
    pcvo_rng br;
    pcvo_rng_init(&br, cfg->seed, pcvo_stream_key(PCVG_STREAM_BENCHMARK, (uint64_t)r, 0, 0));
    double best = -1.0;
    double sx[256], sxx[256];
    for (int m = 0; m < n_models; ++m)
      for (int k = 0; k < K; ++k) {
        if (failed[k]) continue;
        for (int c = 0; c < l; ++c) {
          sx[c] = 0.0;
          sxx[c] = 0.0;
          for (int blk = 0; blk < D; ++blk) {
            const int src = (int)pcvo_below(&br, (uint64_t)l);
            const score_accum* a = &rc.tasks[((long)m * K + k) * l + src].acc;
            sx[c] += a->y_x[blk];
            sxx[c] += a->y_x2[blk];
          }
        }
        double rr;
        if (pcvo_rhat_from_sums(sx, sxx, l, n, NULL, NULL, &rr) && rr > best) best = rr;
      }
    if (best >= 0.0 && rep->benchmark) rep->benchmark[rep->benchmark_count++] = best;
  }
  rep->verdict_quantile = cfg->bench_quantile;
  if (isfinite(rep->rhat_max) && rep->benchmark_count > 0) {
    rep->verdict_quantile_value = pcvo_benchmark_quantile(rep->benchmark, rep->benchmark_count, cfg->bench_quantile);
    rep->verdict_observed = rep->rhat_max;
    rep->verdict_pass = rep->rhat_max <= rep->verdict_quantile_value;
  } else {
    rep->verdict_pass = 1;
    rep->verdict_quantile_value = NAN;
    rep->verdict_observed = rep->rhat_max;
  }
  rep->iters_run = n;
  if (tout) {
    const int stride = 10 + 2 * D;
    for (long i = 0; i < rc.n_tasks; ++i) {
      const chain_task* t = &rc.tasks[i];
      if (tout->position) memcpy(tout->position + i * dim_max, t->position, sizeof(double) * models[t->model]->dim);
      if (tout->warm_logpred) tout->warm_logpred[i] = t->warm_logpred;
      if (tout->divergences) tout->divergences[i] = t->sampling_divergences;
      if (tout->accum) {
        double* a = tout->accum + i * stride;
        a[0] = t->acc.u_x; a[1] = t->acc.u_x2; a[2] = t->acc.z_x; a[3] = t->acc.v_x; a[4] = t->acc.v_x2;
        a[5] = (double)t->acc.committed; a[6] = t->acc.pending; a[7] = (double)t->acc.count;
        a[8] = (double)t->acc.faults; a[9] = t->acc.c;
        for (int d = 0; d < D; ++d) { a[10 + d] = t->acc.y_x[d]; a[10 + D + d] = t->acc.y_x2[d]; }
      }
    }
  }
  for (long i = 0; i < rc.n_tasks; ++i) {
    chain_task* t = &rc.tasks[i];
    free(t->position); free(t->snaps);
    if (t->x_snaps) {
      for (int ci = 0; ci < rc.n_ckpt; ++ci) free(t->x_snaps[ci]);
      free(t->x_snaps); free(t->x_acc); free(t->x_warm);
    }
  }
  for (int m = 0; m < n_models; ++m) free(rc.centers[m]);
  if (rc.x_centers) {
    for (int m = 0; m < n_models; ++m) {
      for (int k = 0; k < K; ++k) free(rc.x_centers[m][k]);
      free(rc.x_centers[m]);
    }
    free(rc.x_centers);
  }
  free(rc.centers); free(rc.tasks); free(rc.checkpoints); free(failed); free(fs); free(rh); free(fl); free(rg);
  return 0;
}

/* ------------------------------------------------------------------ bench sampler timing
 * Steps 2-3 task loop (engine.cpp:296-381) on a fold sample, `threads` pthreads; the C-port CPU
 * baseline when the reference build is absent. */
typedef struct {
  const pcvo_model* m;
  const int32_t* folds;
  int32_t L;
  int64_t warmup, iters;
  uint64_t seed;
  int32_t model_id;
  const pcvg_kernel* k;
  const double* bank;
  int64_t bank_rows;
  long ntask;
  atomic_long next;
  double* pos;  /* [ntask*dim] */
  pcvo_rng* rng;
  double* warm;
  score_accum* acc;
  int phase;
} time_ctx;

static void* time_worker(void* arg) {
  time_ctx* tc = arg;
  const int d = tc->m->dim;
  double* mom = malloc(sizeof(double) * d);
  double* wq = malloc(sizeof(double) * d);
  double* wp = malloc(sizeof(double) * d);
  for (;;) {
    const long i = atomic_fetch_add(&tc->next, 1);
    if (i >= tc->ntask) break;
    const int fold = tc->folds[i / tc->L], chain = (int)(i % tc->L);
    double* pos = tc->pos + i * d;
    int32_t acc;
    if (tc->phase == 2) {
      pcvo_rng init;
      pcvo_rng_init(&init, tc->seed, pcvo_stream_key(PCVG_STREAM_CHAIN_INIT, (uint64_t)tc->model_id, (uint64_t)fold, (uint64_t)chain));
      const uint64_t row = pcvo_below(&init, (uint64_t)tc->bank_rows);
      memcpy(pos, tc->bank + row * d, sizeof(double) * d);
      pcvo_rng_init(&tc->rng[i], tc->seed, pcvo_stream_key(PCVG_STREAM_CHAIN_SAMPLING, (uint64_t)tc->model_id, (uint64_t)fold, (uint64_t)chain));
      tc->warm[i] = 0.0;
      for (int64_t s = 0; s < tc->warmup; ++s) {
        hmc_step_rng(tc->m, fold, tc->k->step_size, tc->k->n_leapfrog, tc->k->inv_mass_diag, pos, &tc->rng[i], mom, wq, wp, &acc);
        tc->warm[i] += pcvo_log_pred(tc->m, pos, fold);
      }
    } else {
      const double c = tc->warmup > 0 ? tc->warm[i] / ((double)tc->L * tc->warmup) : 0.0;
      accum_init(&tc->acc[i], tc->iters < 50 ? (int)tc->iters : 50, 5, tc->iters, c);
      for (int64_t s = 0; s < tc->iters; ++s) {
        hmc_step_rng(tc->m, fold, tc->k->step_size, tc->k->n_leapfrog, tc->k->inv_mass_diag, pos, &tc->rng[i], mom, wq, wp, &acc);
        accum_observe(&tc->acc[i], pcvo_log_pred(tc->m, pos, fold), s);
      }
    }
  }
  free(mom); free(wq); free(wp);
  return NULL;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

int pcvo_time_tasks(const pcvo_model* m, int32_t n_folds, const int32_t* folds, int32_t L,
                    int64_t warmup, int64_t iters, uint64_t seed, int32_t model_id,
                    const pcvg_kernel* k, const double* bank, int64_t bank_rows, int32_t threads,
                    double* sampling_s, double* warmup_s, double* checksum) {
  time_ctx tc;
  memset(&tc, 0, sizeof tc);
  tc.m = m; tc.folds = folds; tc.L = L; tc.warmup = warmup; tc.iters = iters; tc.seed = seed;
  tc.model_id = model_id; tc.k = k; tc.bank = bank; tc.bank_rows = bank_rows;
  tc.ntask = (long)n_folds * L;
  tc.pos = malloc(sizeof(double) * tc.ntask * m->dim);
  tc.rng = malloc(sizeof(pcvo_rng) * tc.ntask);
  tc.warm = malloc(sizeof(double) * tc.ntask);
  tc.acc = malloc(sizeof(score_accum) * tc.ntask);
  if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  double t[3];
  t[0] = now_s();
  for (int phase = 2; phase <= 3; ++phase) {
    tc.phase = phase;
    atomic_store(&tc.next, 0);
    pthread_t* th = malloc(sizeof(pthread_t) * threads);
    for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, time_worker, &tc);
    for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    free(th);
    t[phase - 1] = now_s();
  }
  *warmup_s = t[1] - t[0];
  *sampling_s = t[2] - t[1];
  double cs = 0.0;
  for (long i = 0; i < tc.ntask; ++i) cs += tc.acc[i].u_x;
  *checksum = cs;
  free(tc.pos); free(tc.rng); free(tc.warm); free(tc.acc);
  return 0;
}

/* ------------------------------------------------------------------ accumulator probe
 * Feeds L chains' score streams (stream c = s[c*n .. c*n+n)) through ScoreAccum::observe
 * (accum.cpp:164-182) and reduces them with logs_fold_score + rhat_from_blocks
 * (scoring.cpp:10-62, diagnostics.cpp:35-44). out: estimate, log_f_hat, mc, naive, ess, rhat,
 * batches, fault. */
int pcvo_score_streams(int32_t L, int64_t n, const double* s, double center, int32_t b, int32_t D,
                       double* out) {
  if (L < 1 || L > 256 || n < 1 || D < 1 || D > 16 || b < 1) return set_err(PCVG_INVALID_INPUT, "bad stream probe");
  score_accum* a = malloc(sizeof(score_accum) * L);
  const score_accum* ch[256];
  for (int c = 0; c < L; ++c) {
    accum_init(&a[c], b, D, n, center);
    for (int64_t i = 0; i < n; ++i) accum_observe(&a[c], s[c * n + i], i);
    ch[c] = &a[c];
  }
  const fold_score fs = logs_fold_score(ch, L, n);
  double rh;
  const int ok = rhat_from_blocks(ch, L, n, &rh);
  out[0] = fs.estimate; out[1] = fs.log_f_hat; out[2] = fs.mc; out[3] = fs.naive; out[4] = fs.ess;
  out[5] = ok ? rh : NAN; out[6] = (double)fs.batches; out[7] = fs.fault;
  free(a);
  return 0;
}
