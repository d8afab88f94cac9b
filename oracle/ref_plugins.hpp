// TEST INFRASTRUCTURE ONLY (oracle). Two model plugins written against the
// reference's own plugin API `pcv::Model` (/root/reference/proj/include/pcv/model.hpp:24-78)
// so that the reference engine `pcv::run_pcv` (src/engine.cpp:257-483) can run the two
// BASELINE configs the reference does not ship:
//
//  * LogisticModel  - cfg2 (BASELINE.json configs[1]). New family: the reference has no
//    non-Gaussian likelihood. Written from scratch following the Model
//    conventions: unconstrained parameters, masked training sum `mask * term`
//    (grouped_regression.cpp:174-177), fold K = full-data sentinel (model.hpp:17-20).
//  * HvSeasonalARModel - cfg4 hv-block folds. The reference's FoldAssignment is a partition
//    (folds.hpp:10-20) and cannot express a gap h; this plugin delegates every evaluation to
//    unmodified reference `SeasonalARModel` instances built on two-way partitions
//    ({excluded rows, rest} for log_joint/grad, {test rows, rest} for log_pred), so the
//    per-observation arithmetic stays the reference's own (seasonal_ar.cpp:59-115).
//
// Nothing under oracle/ is linked into the product (paper_2310_07002_b200/).
#pragma once

#include <memory>
#include <vector>

#include "pcv/dataset.hpp"
#include "pcv/folds.hpp"
#include "pcv/model.hpp"
#include "pcv/models/seasonal_ar.hpp"

namespace pcvoracle {

// y_i ~ Bernoulli(sigmoid(beta_0 + sum_p x_ip beta_p)), beta_j ~ N(0, 1).
// Layout: [beta_0 (intercept), beta_1..beta_P].
class LogisticModel : public pcv::Model {
 public:
  LogisticModel(std::string name, pcv::Dataset data, pcv::FoldAssignment folds);
  std::string name() const override { return name_; }
  int dim() const override { return p_ + 1; }
  int fold_count() const override { return folds_.K; }
  long test_size(int fold_id) const override { return folds_.test_size(fold_id); }
  double log_joint(std::span<const double> theta, int fold_id) const override;
  void grad_log_joint(std::span<const double> theta, int fold_id,
                      std::span<double> grad) const override;
  double log_pred(std::span<const double> theta, int fold_id) const override;
  double log_lik_test(std::span<const double> theta, int fold_id) const override;
  std::vector<double> initial_draw(pcv::CounterRng& rng) const override;
  std::vector<double> test_values(int fold_id) const override;

  double eta(std::span<const double> theta, long obs) const;

 private:
  int p_;
  std::string name_;
  pcv::Dataset data_;
  pcv::FoldAssignment folds_;
  std::vector<std::vector<int>> test_obs_;
};

// hv-block fold k (time-rank space): test rows rank in [test_lo, test_hi); training rows
// rank outside [ex_lo, ex_hi) with ex_lo <= test_lo < test_hi <= ex_hi.
struct HvFold {
  long test_lo, test_hi, ex_lo, ex_hi;
};

class HvSeasonalARModel : public pcv::Model {
 public:
  HvSeasonalARModel(std::string name, const pcv::Dataset& data, std::vector<HvFold> folds,
                    int ar_order, int dummies, pcv::RhoTransform tf);
  std::string name() const override { return name_; }
  int dim() const override { return full_->dim(); }
  int fold_count() const override { return static_cast<int>(folds_.size()); }
  long test_size(int fold_id) const override;
  double log_joint(std::span<const double> theta, int fold_id) const override;
  void grad_log_joint(std::span<const double> theta, int fold_id,
                      std::span<double> grad) const override;
  double log_pred(std::span<const double> theta, int fold_id) const override;
  double log_lik_test(std::span<const double> theta, int fold_id) const override;
  std::vector<double> initial_draw(pcv::CounterRng& rng) const override {
    return full_->initial_draw(rng);
  }
  std::vector<double> test_values(int fold_id) const override;
  // HS / DSS hooks: the unmodified SeasonalARModel on the fold's test partition
  // (seasonal_ar.cpp:133-150), test rows in time order as log_pred uses them.
  bool supports_pred_derivs() const override { return true; }
  void pred_derivs(std::span<const double> theta, int fold_id, std::span<double> d1,
                   std::span<double> d2) const override {
    test_[fold_id]->pred_derivs(theta, 0, d1, d2);
  }
  bool supports_pred_sample() const override { return true; }
  void pred_sample(std::span<const double> theta, int fold_id, pcv::CounterRng& rng,
                   std::span<double> out) const override {
    test_[fold_id]->pred_sample(theta, 0, rng, out);
  }

 private:
  std::string name_;
  std::vector<HvFold> folds_;
  std::vector<long> rank_;  // time rank of each row
  // train_[k]: partition {0: excluded rows, 1: rest}; test_[k]: {0: test rows, 1: rest}.
  std::vector<std::unique_ptr<pcv::SeasonalARModel>> train_, test_;
  std::unique_ptr<pcv::SeasonalARModel> full_;  // sentinel evaluations
};

}  // namespace pcvoracle
