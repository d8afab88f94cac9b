// Fold schemes and simulators (host, bit-exact with the reference where it has them).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "../../include/pcvg.h"
#include "host_common.hpp"

namespace pcvg {

std::vector<int64_t> time_order(const int64_t* t, int64_t n) {
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return t[a] < t[b]; });
  return order;
}

namespace {

void check_dataset(const pcvg_dataset* d) {  // Dataset::validate, dataset.cpp:19-39
  if (!d || d->n_obs < 1) throw Error(PCVG_INVALID_INPUT, "dataset is empty");
  if (d->n_cov < 0 || (d->n_cov > 0 && !d->x)) throw Error(PCVG_INVALID_INPUT, "covariate matrix size does not match n_obs");
  if (d->group_id) {
    int32_t j = 0;
    for (int64_t i = 0; i < d->n_obs; ++i) j = std::max(j, d->group_id[i] + 1);
    std::vector<char> seen(j, 0);
    for (int64_t i = 0; i < d->n_obs; ++i) {
      if (d->group_id[i] < 0) throw Error(PCVG_INVALID_INPUT, "group ids must be 0-based");
      seen[d->group_id[i]] = 1;
    }
    for (int g = 0; g < j; ++g)
      if (!seen[g]) throw Error(PCVG_INVALID_INPUT, "group ids must form a contiguous 0..J-1 range");
  }
}

}  // namespace
}  // namespace pcvg

using pcvg::Error;
using pcvg::HostRng;

extern "C" {

uint64_t pcvg_stream_key(uint64_t kind, uint64_t a, uint64_t b, uint64_t c) {
  return pcvg::stream_key(kind, a, b, c);
}

}  // extern "C"

// Exported through api.cpp's error-mapping wrapper.
namespace pcvg {

void rng_sequence(uint64_t seed, uint64_t stream, int32_t do_skip, uint64_t skip_block,
                  const char* ops, const uint64_t* arg, int64_t n, double* out) {
  HostRng r(seed, stream);
  if (do_skip) r.skip_to(skip_block);
  for (int64_t i = 0; i < n; ++i) {
    switch (ops[i]) {
      case 'u': out[i] = r.uniform(); break;
      case 'n': out[i] = r.normal(); break;
      case '4': out[i] = static_cast<double>(r.next_u32()); break;
      case 'b':
        if (arg[i] == 0) throw Error(PCVG_INVALID_INPUT, "below(0)");
        out[i] = static_cast<double>(r.below(arg[i]));
        break;
      default: throw Error(PCVG_INVALID_INPUT, "bad rng op");
    }
  }
}

void make_loo(int64_t n, int32_t* ti, int32_t* K) {  // folds.cpp:43-52
  if (n < 2) throw Error(PCVG_INVALID_INPUT, "LOO needs at least 2 observations");
  for (int64_t i = 0; i < n; ++i) ti[i] = static_cast<int32_t>(i);
  *K = static_cast<int32_t>(n);
}

void make_logo(const pcvg_dataset* d, int32_t* ti, int32_t* K) {  // folds.cpp:54-63
  if (!d->group_id) throw Error(PCVG_INVALID_INPUT, "LOGO requires a group column");
  check_dataset(d);
  int32_t j = 0;
  for (int64_t i = 0; i < d->n_obs; ++i) j = std::max(j, d->group_id[i] + 1);
  if (j < 2) throw Error(PCVG_INVALID_INPUT, "fold 0 has empty training set");
  std::memcpy(ti, d->group_id, sizeof(int32_t) * d->n_obs);
  *K = j;
}

void make_kfold(int64_t n, int32_t K, uint64_t seed, int32_t* ti) {  // folds.cpp:65-84
  if (K < 2 || K > n) throw Error(PCVG_INVALID_INPUT, "K-fold requires 2 <= K <= n_obs");
  const int64_t base = n / K, rem = n % K;
  int64_t pos = 0;
  for (int k = 0; k < K; ++k)
    for (int64_t i = 0; i < base + (k < rem ? 1 : 0); ++i) ti[pos++] = k;
  HostRng rng(seed, stream_key(PCVG_STREAM_KFOLD, static_cast<uint64_t>(K), 0, 0));
  for (int64_t i = n - 1; i > 0; --i) std::swap(ti[i], ti[rng.below(i + 1)]);
}

void make_time_blocks(const pcvg_dataset* d, int32_t K, int32_t* ti) {  // folds.cpp:86-108
  const int64_t n = d->n_obs;
  if (!d->time_index) throw Error(PCVG_INVALID_INPUT, "time-block scheme requires a time column");
  if (K < 2 || K > n) throw Error(PCVG_INVALID_INPUT, "time-block scheme requires 2 <= K <= n_obs");
  const auto order = time_order(d->time_index, n);
  const int64_t base = n / K, rem = n % K;
  int64_t pos = 0;
  for (int k = 0; k < K; ++k) {
    const int64_t len = base + (k < rem ? 1 : 0);
    for (int64_t i = 0; i < len; ++i) ti[order[pos++]] = k;
  }
}

// hv-block (Racine 2000; new - SPEC.md:114 left it unimplemented): the time-block test partition
// (sizes as folds.cpp:99-106) with h ranks on each side also removed from training.
void make_hv_block(const pcvg_dataset* d, int32_t K, int64_t h, int64_t* iv) {
  const int64_t n = d->n_obs;
  if (!d->time_index) throw Error(PCVG_INVALID_INPUT, "hv-block requires a time column");
  if (K < 2 || K > n || h < 0) throw Error(PCVG_INVALID_INPUT, "hv-block requires 2 <= K <= n_obs and h >= 0");
  const int64_t base = n / K, rem = n % K;
  int64_t pos = 0;
  for (int k = 0; k < K; ++k) {
    const int64_t len = base + (k < rem ? 1 : 0);
    iv[4 * k] = pos;
    iv[4 * k + 1] = pos + len;
    iv[4 * k + 2] = std::max<int64_t>(0, pos - h);
    iv[4 * k + 3] = std::min<int64_t>(n, pos + len + h);
    if (iv[4 * k + 3] - iv[4 * k + 2] >= n) throw Error(PCVG_INVALID_INPUT, "hv-block fold has empty training set");
    pos += len;
  }
}

void make_hv_racine(const pcvg_dataset* d, int64_t v, int64_t h, int64_t* iv) {
  const int64_t n = d->n_obs;
  if (!d->time_index) throw Error(PCVG_INVALID_INPUT, "hv-block requires a time column");
  if (v < 0 || h < 0) throw Error(PCVG_INVALID_INPUT, "hv-block requires v, h >= 0");
  for (int64_t t = 0; t < n; ++t) {
    iv[4 * t] = std::max<int64_t>(0, t - v);
    iv[4 * t + 1] = std::min<int64_t>(n, t + v + 1);
    iv[4 * t + 2] = std::max<int64_t>(0, t - v - h);
    iv[4 * t + 3] = std::min<int64_t>(n, t + v + h + 1);
    if (iv[4 * t + 3] - iv[4 * t + 2] >= n) throw Error(PCVG_INVALID_INPUT, "hv-block fold has empty training set");
  }
}

// simulate_grouped_regression, grouped_regression.cpp:232-268.
void simulate_grouped(int32_t J, int32_t Nj, int32_t P, double min_beta, uint64_t seed, double* y,
                      double* x, int32_t* g, SimTruth* truth) {
  if (J < 2) throw Error(PCVG_INVALID_INPUT, "simulator needs at least 2 groups");
  if (Nj < 1 || P < 1) throw Error(PCVG_INVALID_INPUT, "simulator needs per_group and covariates >= 1");
  HostRng rng(seed, stream_key(PCVG_STREAM_SIMULATE, 1, 0, 0));
  const double mu_alpha = rng.normal();
  const double sigma_alpha = std::fabs(rng.normal()) * std::sqrt(10.0);
  const double sigma_y = std::fabs(rng.normal()) * std::sqrt(10.0);
  std::vector<double> beta(P);
  for (double& b : beta) b = rng.normal();
  if (min_beta > 0.0)
    while (std::fabs(beta.back()) < min_beta) beta.back() = rng.normal();
  std::vector<double> alpha(J);
  for (double& a : alpha) a = mu_alpha + sigma_alpha * rng.normal();
  std::vector<double> xg(static_cast<size_t>(J) * P);
  for (double& v : xg) v = rng.normal() * std::sqrt(10.0);
  int64_t row = 0;
  for (int gg = 0; gg < J; ++gg)
    for (int i = 0; i < Nj; ++i, ++row) {
      double mean = alpha[gg];
      for (int p = 0; p < P; ++p) mean += xg[gg * P + p] * beta[p];
      y[row] = mean + sigma_y * rng.normal();
      for (int p = 0; p < P; ++p) x[row * P + p] = xg[gg * P + p];
      g[row] = gg;
    }
  if (truth) {
    truth->vectors = {{"alpha", alpha}, {"beta", beta}};
    truth->scalars = {{"mu_alpha", mu_alpha}, {"sigma_alpha", sigma_alpha}, {"sigma_y", sigma_y}};
  }
}

// simulate_radon_style, radon.cpp:216-240.
// simulate_rat_growth (rat_growth.cpp:310-336): n = 5 * subjects at times {8,15,22,29,36}.
void simulate_rat(int32_t subjects, uint64_t seed, double* y, double* x, int32_t* g, SimTruth* truth) {
  if (subjects < 2) throw Error(PCVG_INVALID_INPUT, "simulator needs at least 2 subjects");
  HostRng rng(seed, stream_key(PCVG_STREAM_SIMULATE, 2, 0, 0));
  const double mu_alpha = 250.0 + std::sqrt(20.0) * rng.normal();
  const double mu_beta = 6.0 + std::sqrt(2.0) * rng.normal();
  const double sigma_alpha = gamma_draw(rng, 25.0, 2.0);
  const double sigma_beta = gamma_draw(rng, 5.0, 10.0);
  const double sigma_y = gamma_draw(rng, 1.0, 2.0);
  const double times[5] = {8, 15, 22, 29, 36};
  int64_t i = 0;
  std::vector<double> alpha, beta;
  for (int s = 0; s < subjects; ++s) {
    const double a = mu_alpha + sigma_alpha * rng.normal();
    const double b = mu_beta + sigma_beta * rng.normal();
    alpha.push_back(a);
    beta.push_back(b);
    for (double t : times) {
      y[i] = a + b * t + sigma_y * rng.normal();
      x[i] = t;
      g[i] = s;
      ++i;
    }
  }
  if (truth) {
    truth->vectors = {{"alpha", alpha}, {"beta", beta}};
    truth->scalars = {{"mu_alpha", mu_alpha}, {"mu_beta", mu_beta}, {"sigma_alpha", sigma_alpha},
                      {"sigma_beta", sigma_beta}, {"sigma_y", sigma_y}};
  }
}

void simulate_radon(int32_t houses, int32_t counties, uint64_t seed, double* y, double* x,
                    int32_t* g, SimTruth* truth) {
  if (counties < 2 || houses < counties)
    throw Error(PCVG_INVALID_INPUT, "simulator needs counties >= 2 and houses >= counties");
  HostRng rng(seed, stream_key(PCVG_STREAM_SIMULATE, 3, 0, 0));
  const double mu_alpha = 2.0 * rng.normal();
  const double sigma_alpha2 = gamma_draw(rng, 6.0, 9.0);
  const double sigma_y2 = gamma_draw(rng, 10.0, 10.0);
  const double beta = rng.normal();
  std::vector<double> alpha(counties);
  for (int c = 0; c < counties; ++c) alpha[c] = mu_alpha + std::sqrt(sigma_alpha2) * rng.normal();
  for (int i = 0; i < houses; ++i) {
    const int gg = i % counties;
    const double floor = rng.uniform() < 0.5 ? 0.0 : 1.0;
    y[i] = alpha[gg] + beta * floor + std::sqrt(sigma_y2) * rng.normal();
    x[i] = floor;
    g[i] = gg;
  }
  if (truth) {
    truth->vectors = {{"alpha", alpha}};
    truth->scalars = {{"beta", beta}, {"mu_alpha", mu_alpha}, {"sigma_alpha2", sigma_alpha2},
                      {"sigma_y2", sigma_y2}};
  }
}

// simulate_seasonal_ar, seasonal_ar.cpp:167-205.
void simulate_seasonal(int64_t months, int32_t p, int32_t q, double rho, double amp, double sigma,
                       uint64_t seed, double* y, double* x, int64_t* t, SimTruth* truth) {
  if (months <= p + q) throw Error(PCVG_INVALID_INPUT, "series too short for the requested AR order and dummies");
  if (p < 1) throw Error(PCVG_INVALID_INPUT, "AR order must be at least 1");
  HostRng rng(seed, stream_key(PCVG_STREAM_SIMULATE, 4, 0, 0));
  std::vector<double> rhos(p, 0.0), beta(q + 1, 0.0);
  rhos[0] = rho;
  for (int j = 1; j <= q; ++j) beta[j] = amp * rng.normal();
  std::vector<double> series(months, 0.0);
  for (int64_t s = 0; s < months; ++s) {
    double m = beta[0];
    for (int i = 0; i < p; ++i)
      if (s - 1 - i >= 0) m += rhos[i] * series[s - 1 - i];
    const int month = static_cast<int>(s % 12);
    if (month >= 1 && month <= q) m += beta[month];
    series[s] = m + sigma * rng.normal();
  }
  const int nc = p + q;
  int64_t row = 0;
  for (int64_t s = p; s < months; ++s, ++row) {
    y[row] = series[s];
    for (int i = 0; i < p; ++i) x[row * nc + i] = series[s - 1 - i];
    const int month = static_cast<int>(s % 12);
    for (int j = 1; j <= q; ++j) x[row * nc + p + j - 1] = month == j ? 1.0 : 0.0;
    t[row] = s;
  }
  if (truth) {
    truth->vectors = {{"beta", beta}, {"rho", rhos}};
    truth->scalars = {{"sigma", sigma}};
  }
}

// cfg1 / cfg5 linear regression (new shape; grouped family with J = 1).
void simulate_linreg(int64_t n, int32_t P, uint64_t seed, double* y, double* x, int32_t* g) {
  if (n < 2 || P < 1) throw Error(PCVG_INVALID_INPUT, "linreg simulator needs n >= 2, P >= 1");
  HostRng rng(seed, stream_key(PCVG_STREAM_SIMULATE, 6, 0, 0));
  for (int64_t i = 0; i < n; ++i) {
    double m = 0.5;
    for (int p = 0; p < P; ++p) {
      x[i * P + p] = rng.normal();
      m += 0.3 * (p + 1) * x[i * P + p];
    }
    y[i] = m + rng.normal();
    if (g) g[i] = 0;
  }
}

// cfg2 logistic regression (new family).
void simulate_logistic(int64_t n, int32_t P, uint64_t seed, double* y, double* x) {
  if (n < 2 || P < 1) throw Error(PCVG_INVALID_INPUT, "logistic simulator needs n >= 2, P >= 1");
  HostRng rng(seed, stream_key(PCVG_STREAM_SIMULATE, 5, 0, 0));
  std::vector<double> beta(P + 1);
  for (double& b : beta) b = rng.normal();
  const double scale = 1.0 / std::sqrt(static_cast<double>(P));
  for (int64_t i = 0; i < n; ++i) {
    double eta = beta[0];
    for (int p = 0; p < P; ++p) {
      x[i * P + p] = rng.normal() * scale;
      eta += x[i * P + p] * beta[1 + p];
    }
    const double prob = 1.0 / (1.0 + std::exp(-eta));
    y[i] = rng.uniform() < prob ? 1.0 : 0.0;
  }
}

}  // namespace pcvg
