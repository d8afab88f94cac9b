// TEST INFRASTRUCTURE ONLY (oracle). See ref_plugins.hpp.
#include "ref_plugins.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

#include "pcv/errors.hpp"
#include "pcv/math.hpp"

namespace pcvoracle {

namespace {

// log(1 + e^t) without overflow.
double softplus(double t) { return std::max(t, 0.0) + std::log1p(std::exp(-std::fabs(t))); }

double sigmoid(double t) {
  if (t >= 0.0) return 1.0 / (1.0 + std::exp(-t));
  const double e = std::exp(t);
  return e / (1.0 + e);
}

// Bernoulli log mass of y in {0,1} at logit t: y t - log(1 + e^t).
double bernoulli_logit_lpmf(double y, double t) { return y * t - softplus(t); }

}  // namespace

LogisticModel::LogisticModel(std::string name, pcv::Dataset data, pcv::FoldAssignment folds)
    : name_(std::move(name)), data_(std::move(data)), folds_(std::move(folds)) {
  data_.validate();
  folds_.validate(data_.n_obs());
  p_ = data_.n_cov;
  test_obs_.resize(folds_.K);
  for (long i = 0; i < data_.n_obs(); ++i)
    test_obs_[folds_.test_index[i]].push_back(static_cast<int>(i));
}

double LogisticModel::eta(std::span<const double> theta, long obs) const {
  double t = theta[0];
  for (int p = 0; p < p_; ++p) t += data_.xv(obs, p) * theta[1 + p];
  return t;
}

double LogisticModel::log_joint(std::span<const double> theta, int fold_id) const {
  double lp = 0.0;
  for (long i = 0; i < data_.n_obs(); ++i) {
    const double mask = folds_.test_index[i] == fold_id ? 0.0 : 1.0;
    lp += mask * bernoulli_logit_lpmf(data_.y[i], eta(theta, i));
  }
  for (int j = 0; j <= p_; ++j) lp += pcv::normal_logpdf(theta[j], 0.0, 1.0);
  return lp;
}

void LogisticModel::grad_log_joint(std::span<const double> theta, int fold_id,
                                   std::span<double> grad) const {
  for (int j = 0; j <= p_; ++j) grad[j] = 0.0;
  for (long i = 0; i < data_.n_obs(); ++i) {
    if (folds_.test_index[i] == fold_id) continue;
    const double r = data_.y[i] - sigmoid(eta(theta, i));
    grad[0] += r;
    for (int p = 0; p < p_; ++p) grad[1 + p] += data_.xv(i, p) * r;
  }
  for (int j = 0; j <= p_; ++j) grad[j] -= theta[j];
}

double LogisticModel::log_pred(std::span<const double> theta, int fold_id) const {
  if (fold_id >= folds_.K) return 0.0;
  double lp = 0.0;
  for (int i : test_obs_[fold_id]) lp += bernoulli_logit_lpmf(data_.y[i], eta(theta, i));
  return lp;
}

double LogisticModel::log_lik_test(std::span<const double> theta, int fold_id) const {
  return log_pred(theta, fold_id);
}

std::vector<double> LogisticModel::initial_draw(pcv::CounterRng& rng) const {
  std::vector<double> theta(dim());
  for (double& t : theta) t = rng.normal();
  return theta;
}

std::vector<double> LogisticModel::test_values(int fold_id) const {
  std::vector<double> y;
  for (int i : test_obs_[fold_id]) y.push_back(data_.y[i]);
  return y;
}

HvSeasonalARModel::HvSeasonalARModel(std::string name, const pcv::Dataset& data,
                                     std::vector<HvFold> folds, int ar_order, int dummies,
                                     pcv::RhoTransform tf)
    : name_(std::move(name)), folds_(std::move(folds)) {
  const long n = data.n_obs();
  if (!data.has_time()) throw pcv::invalid_input("hv-block needs a time column");
  std::vector<long> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](long a, long b) {
    return data.time_index[a] < data.time_index[b];
  });
  rank_.assign(n, 0);
  for (long r = 0; r < n; ++r) rank_[order[r]] = r;

  auto two_way = [&](long lo, long hi) {
    pcv::FoldAssignment f;
    f.K = 2;
    f.test_index.assign(n, 1);
    for (long i = 0; i < n; ++i)
      if (rank_[i] >= lo && rank_[i] < hi) f.test_index[i] = 0;
    return f;
  };
  for (const HvFold& hf : folds_) {
    train_.push_back(std::make_unique<pcv::SeasonalARModel>(
        name_, data, two_way(hf.ex_lo, hf.ex_hi), ar_order, dummies, tf));
    test_.push_back(std::make_unique<pcv::SeasonalARModel>(
        name_, data, two_way(hf.test_lo, hf.test_hi), ar_order, dummies, tf));
  }
  full_ = std::make_unique<pcv::SeasonalARModel>(name_, data, two_way(0, 1), ar_order,
                                                 dummies, tf);
}

long HvSeasonalARModel::test_size(int fold_id) const {
  if (fold_id >= fold_count()) return 0;
  return folds_[fold_id].test_hi - folds_[fold_id].test_lo;
}

double HvSeasonalARModel::log_joint(std::span<const double> theta, int fold_id) const {
  if (fold_id >= fold_count()) return full_->log_joint(theta, 2);
  return train_[fold_id]->log_joint(theta, 0);
}

void HvSeasonalARModel::grad_log_joint(std::span<const double> theta, int fold_id,
                                       std::span<double> grad) const {
  if (fold_id >= fold_count()) return full_->grad_log_joint(theta, 2, grad);
  train_[fold_id]->grad_log_joint(theta, 0, grad);
}

double HvSeasonalARModel::log_pred(std::span<const double> theta, int fold_id) const {
  if (fold_id >= fold_count()) return 0.0;
  return test_[fold_id]->log_pred(theta, 0);
}

double HvSeasonalARModel::log_lik_test(std::span<const double> theta, int fold_id) const {
  return log_pred(theta, fold_id);
}

std::vector<double> HvSeasonalARModel::test_values(int fold_id) const {
  return test_[fold_id]->test_values(0);
}

}  // namespace pcvoracle
