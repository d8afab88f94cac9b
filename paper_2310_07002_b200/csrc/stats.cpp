// Step 4 on the host: merge the per-fold tables (produced on device, gathered across GPUs in
// fold order) into the global statistics exactly as compute_stats (engine.cpp:117-253), the
// report assembly (engine.cpp:410-459) and the shuffle benchmark / verdict
// (engine.cpp:464-480, diagnostics.cpp:76-119). Fold-order sums keep the result bit-identical for
// any number of GPUs.
#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "../../include/pcvg.h"
#include "host_common.hpp"

namespace pcvg {

namespace {

const double kNaN = std::numeric_limits<double>::quiet_NaN();
const double kInf = std::numeric_limits<double>::infinity();

bool rhat_from_sums(const double* sx, const double* sxx, int l, int64_t n, double* rhat) {
  if (l < 2 || n < 2) return false;  // diagnostics.cpp:11-33
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
  b *= static_cast<double>(n) / (l - 1.0);
  if (!std::isfinite(w) || !std::isfinite(b) || !(w > 0.0)) return false;
  *rhat = std::sqrt(((n - 1.0) / n * w + b / n) / w);
  return true;
}

// Cholesky helpers, math.hpp:46-76 (row-major n x n, lower factor in place).
bool cholesky_in_place(std::vector<double>& a, int n) {
  for (int j = 0; j < n; ++j) {
    double d = a[j * n + j];
    for (int k = 0; k < j; ++k) d -= a[j * n + k] * a[j * n + k];
    if (!(d > 0.0) || !std::isfinite(d)) return false;
    const double l = std::sqrt(d);
    a[j * n + j] = l;
    for (int i = j + 1; i < n; ++i) {
      double s = a[i * n + j];
      for (int k = 0; k < j; ++k) s -= a[i * n + k] * a[j * n + k];
      a[i * n + j] = s / l;
    }
  }
  return true;
}

}  // namespace

// hs_fold_score (scoring.cpp:64-73) on the chain-merged WelfordDiag of xi = (d2 + d1^2, d1):
// mu = a_x / count + c; the report carries the negation (engine.cpp:157-158).
double hs_fold_estimate(const double* a_x, const double* center, int m, int64_t count) {
  double score = 0.0;
  for (int i = 0; i < m; ++i) {
    const double mu1 = a_x[i] / static_cast<double>(count) + center[i];
    const double mu2 = a_x[m + i] / static_cast<double>(count) + center[m + i];
    score += 2.0 * mu1 - mu2 * mu2;
  }
  return -score;
}

// dss_fold_score (scoring.cpp:75-104) on the chain-merged WelfordAccumulator (a_x[m], packed lower
// triangle a_xx): mean / covariance as WelfordAccumulator::mean/covariance (accum.cpp:36-57), a
// ridge of 1e-8 tr/m on a failed factorisation. Returns false where the reference throws
// (too few draws, singular covariance): the fold becomes NaN + fault (engine.cpp:162-170).
bool dss_fold_estimate(const double* merged, const double* center, const double* y_test, int m,
                       int64_t count, double* score, int* ridged) {
  *ridged = 0;
  if (count < m + 1) return false;
  if (count < 2) return false;
  const double* a_x = merged;
  const double* a_xx = merged + m;
  std::vector<double> mu(m), cov(static_cast<size_t>(m) * m);
  for (int i = 0; i < m; ++i) mu[i] = a_x[i] / count + center[i];
  const double inv_n = 1.0 / static_cast<double>(count);
  const double inv_nm1 = 1.0 / static_cast<double>(count - 1);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j <= i; ++j) {
      const double v = (a_xx[static_cast<int64_t>(i) * (i + 1) / 2 + j] - a_x[i] * a_x[j] * inv_n) * inv_nm1;
      cov[i * m + j] = v;
      cov[j * m + i] = v;
    }
  std::vector<double> factor = cov;
  if (!cholesky_in_place(factor, m)) {
    double tr = 0.0;
    for (int i = 0; i < m; ++i) tr += cov[i * m + i];
    const double ridge = 1e-8 * tr / m;
    for (int i = 0; i < m; ++i) cov[i * m + i] += ridge;
    factor = cov;
    *ridged = 1;
    if (!cholesky_in_place(factor, m)) return false;
  }
  std::vector<double> r(m);
  for (int i = 0; i < m; ++i) r[i] = y_test[i] - mu[i];
  for (int i = 0; i < m; ++i) {  // forward_solve, math.hpp:63-70
    double s = r[i];
    for (int k = 0; k < i; ++k) s -= factor[i * m + k] * r[k];
    r[i] = s / factor[i * m + i];
  }
  double quad = 0.0;
  for (int i = 0; i < m; ++i) quad += r[i] * r[i];
  double ld = 0.0;  // chol_logdet, math.hpp:72-76
  for (int i = 0; i < m; ++i) ld += std::log(factor[i * m + i]);
  *score = -(2.0 * ld) - quad;
  return true;
}

// Positional shuffle benchmark of one shard (the host restatement of bench_kernel,
// chain_kernels.cu): y_x / y_x2 are the shard's sub-block sums [m][k][c][D_stride], of which the
// first sub_used are regrouped into `groups` benchmark blocks (block_group_begin); item index of
// (m, local non-failed fold j) = m * nonfailed_total + nonfailed_before + j. rep_max[r] is the max
// R-hat over the shard's items (0 = none); needs_host[r] = 1 on a below() rejection.
void bench_shard(int32_t nm, int32_t nfold, int32_t l, int32_t D_stride, int32_t sub_used, int32_t groups,
                 int64_t n, uint64_t seed, int32_t R, const double* y_x, const double* y_x2,
                 const int32_t* failed, int64_t nonfailed_before, int64_t nonfailed_total,
                 double* rep_max, int32_t* needs_host) {
  const uint64_t L64 = static_cast<uint64_t>(l);
  const uint64_t bound = L64 * ((~uint64_t{0}) / L64);
  std::vector<double> sx(l), sxx(l);
  for (int r = 0; r < R; ++r) {
    rep_max[r] = 0.0;
    needs_host[r] = 0;
    const uint64_t stream = stream_key(PCVG_STREAM_BENCHMARK, static_cast<uint64_t>(r), 0, 0);
    for (int m = 0; m < nm; ++m) {
      int64_t j = 0;
      for (int k = 0; k < nfold; ++k) {
        if (failed && failed[k]) continue;
        const int64_t item = m * nonfailed_total + nonfailed_before + j++;
        uint64_t word = 2ull * static_cast<uint64_t>(item) * L64 * static_cast<uint64_t>(groups);
        HostRng rng(seed, stream);
        const size_t base = (static_cast<size_t>(m) * nfold + k) * l * D_stride;
        for (int c = 0; c < l; ++c) {
          sx[c] = 0.0;
          sxx[c] = 0.0;
          for (int g = 0; g < groups; ++g, word += 2) {
            rng.skip_to(word >> 2);
            if (word & 2) {
              rng.next_u32();
              rng.next_u32();
            }
            const uint64_t v = rng.next_u64();
            if (v >= bound) needs_host[r] = 1;
            const size_t src = static_cast<size_t>(v % L64);
            double ga = 0.0, gb = 0.0;
            for (int d = block_group_begin(g, sub_used, groups); d < block_group_begin(g + 1, sub_used, groups); ++d) {
              ga += y_x[base + src * D_stride + d];
              gb += y_x2[base + src * D_stride + d];
            }
            sx[c] += ga;
            sxx[c] += gb;
          }
        }
        double rr;
        if (rhat_from_sums(sx.data(), sxx.data(), l, n, &rr)) rep_max[r] = std::max(rep_max[r], rr);
      }
    }
  }
}

// final_checkpoint: 0 = intermediate snapshot (no exclusions), 1 = final (exclusions, per-model
// report, benchmark + verdict), 2 = early-stop probe (no exclusions, benchmark + verdict on the
// first sub_used sub-blocks, regrouped into min(blocks, sub_used) blocks).
void merge_stats(int32_t nm, int32_t K, const pcvg_run_config* cfg, int64_t iter_count,
                 int32_t final_checkpoint, const pcvg_fold_table* ft, const double* y_x,
                 const double* y_x2, int sub_used, pcvg_report* rep, const double* bench_max) {
  const int groups = std::min(cfg->blocks, sub_used);
  const int l = cfg->chains;
  const bool final = final_checkpoint == 1;
  const int D_stride = cfg->early_stop ? static_cast<int>(cfg->iters / cfg->checkpoint_every) : cfg->blocks;
  std::vector<char> failed(K, 0), excluded(K, 0);
  if (final && ft->failed)
    for (int k = 0; k < K; ++k) failed[k] = ft->failed[k] != 0;
  for (int k = 0; k < K; ++k) {  // engine.cpp:145-155
    if (final && failed[k]) excluded[k] = 1;
    if (final)
      for (int m = 0; m < nm; ++m)
        if (std::isnan(ft->estimate[static_cast<size_t>(m) * K + k])) excluded[k] = 1;
  }
  double naive_sum = 0.0, mc_sum = 0.0, best = -1.0;
  bool mc_inf = false;
  for (int m = 0; m < nm; ++m)
    for (int k = 0; k < K; ++k) {
      if (excluded[k]) continue;
      const size_t i = static_cast<size_t>(m) * K + k;
      if (std::isfinite(ft->mc_contribution[i])) {
        mc_sum += ft->mc_contribution[i];
        naive_sum += ft->naive_contribution[i];
      } else {
        mc_inf = true;
      }
      if (std::isfinite(ft->rhat[i])) best = std::max(best, ft->rhat[i]);  // rhat_max
    }
  std::vector<double> included;
  included.reserve(K);
  double delta_hat = 0.0;
  for (int k = 0; k < K; ++k) {
    const double dk = nm == 2 ? ft->estimate[k] - ft->estimate[K + k] : ft->estimate[k];
    if (final && rep->delta_k) rep->delta_k[k] = dk;
    if (!excluded[k]) included.push_back(dk);
  }
  for (double dk : included) delta_hat += dk;
  rep->delta_hat = delta_hat;
  if (included.size() >= 2) {  // selection_probability, scoring.cpp:141-158
    const double kk = static_cast<double>(included.size());
    const double mean = delta_hat / kk;
    double ss = 0.0;
    for (double dk : included) ss += (dk - mean) * (dk - mean);
    const double s2 = ss / (kk - 1.0);
    const double denom = std::sqrt(kk * s2);
    double prob;
    if (denom == 0.0) prob = delta_hat > 0.0 ? 1.0 : (delta_hat < 0.0 ? 0.0 : 0.5);
    else prob = 0.5 * std::erfc(-(delta_hat / denom) * 0.70710678118654752440084436210485);
    rep->sigma2_delta = s2;
    rep->epistemic_se = std::sqrt(kk * s2);
    rep->prob_a_better = nm == 2 ? prob : kNaN;
  } else {
    rep->sigma2_delta = rep->epistemic_se = rep->prob_a_better = kNaN;
  }
  const double ln = static_cast<double>(l) * iter_count;
  // MCSE is defined for LogS only (engine.cpp:229-235)
  rep->mcse = cfg->score != PCVG_SCORE_LOGS ? kNaN : (mc_inf ? kInf : std::sqrt(mc_sum / ln));
  rep->ess_overall = mc_sum > 0.0 ? static_cast<double>(l) * iter_count * naive_sum / mc_sum : kNaN;
  rep->rhat_max = best < 0.0 ? kNaN : best;

  if (final) {
    for (int m = 0; m < nm; ++m) {
      rep->score_total[m] = 0.0;
      rep->numeric_faults[m] = 0;
      rep->rhat_excluded[m] = 0;
      for (int k = 0; k < K; ++k) {
        const size_t i = static_cast<size_t>(m) * K + k;
        if (rep->folds.failed) rep->folds.failed[i] = excluded[k];
        if (!excluded[k]) rep->score_total[m] += ft->estimate[i];
        if (ft->fault[i]) ++rep->numeric_faults[m];
        if (!std::isfinite(ft->rhat[i]) && !excluded[k]) ++rep->rhat_excluded[m];
      }
    }
  }
  if (final_checkpoint == 0) return;
  // shuffle benchmark (diagnostics.cpp:76-101) over non-failed folds, model-major
  rep->benchmark_count = 0;
  const int64_t nbench = iter_count;  // = N for a full run (gather_block_sums(chains, n), engine.cpp:471)
  if (bench_max && rep->benchmark) {  // replicate maxima from the device / sharded benchmark
    for (int r = 0; r < cfg->bench_draws; ++r)
      if (bench_max[r] > 0.0) rep->benchmark[rep->benchmark_count++] = bench_max[r];
  } else if (y_x && y_x2 && rep->benchmark) {
    std::vector<double> sx(l), sxx(l);
    for (int r = 0; r < cfg->bench_draws; ++r) {
      HostRng rng(cfg->seed, stream_key(PCVG_STREAM_BENCHMARK, static_cast<uint64_t>(r), 0, 0));
      double rb = -1.0;
      for (int m = 0; m < nm; ++m)
        for (int k = 0; k < K; ++k) {
          if (failed[k]) continue;
          const size_t base = (static_cast<size_t>(m) * K + k) * l * D_stride;
          for (int c = 0; c < l; ++c) {
            sx[c] = 0.0;
            sxx[c] = 0.0;
            for (int g = 0; g < groups; ++g) {
              const int src = static_cast<int>(rng.below(static_cast<uint64_t>(l)));
              double ga = 0.0, gb = 0.0;
              for (int d = block_group_begin(g, sub_used, groups); d < block_group_begin(g + 1, sub_used, groups); ++d) {
                ga += y_x[base + static_cast<size_t>(src) * D_stride + d];
                gb += y_x2[base + static_cast<size_t>(src) * D_stride + d];
              }
              sx[c] += ga;
              sxx[c] += gb;
            }
          }
          double rr;
          if (rhat_from_sums(sx.data(), sxx.data(), l, nbench, &rr)) rb = std::max(rb, rr);
        }
      if (rb >= 0.0) rep->benchmark[rep->benchmark_count++] = rb;
    }
  }
  rep->verdict_quantile = cfg->bench_quantile;
  if (std::isfinite(rep->rhat_max) && rep->benchmark_count > 0) {  // diagnostics.cpp:103-119
    std::vector<double> s(rep->benchmark, rep->benchmark + rep->benchmark_count);
    std::sort(s.begin(), s.end());
    const int64_t n = static_cast<int64_t>(s.size());
    int64_t rank = static_cast<int64_t>(std::ceil(cfg->bench_quantile * n));
    rank = std::clamp<int64_t>(rank, 1, n);
    rep->verdict_quantile_value = s[rank - 1];
    rep->verdict_observed = rep->rhat_max;
    rep->verdict_pass = rep->rhat_max <= rep->verdict_quantile_value;
  } else {
    rep->verdict_pass = 1;
    rep->verdict_quantile_value = kNaN;
    rep->verdict_observed = rep->rhat_max;
  }
}

}  // namespace pcvg
