// TEST INFRASTRUCTURE ONLY (oracle). C shim over the UNMODIFIED reference library
// (/root/reference/proj/src, compiled in place by oracle/Makefile into oracle/_ref/).
// It lets pytest (ctypes) call the reference's own code: RNG (rng.hpp), fold schemes
// (folds.cpp), simulators, Model evaluations (model.hpp:24-78), leapfrog / hmc_step
// (hmc.cpp), adapt_full_data (adapt.cpp) and run_pcv (engine.cpp). It is the checker
// the C restatement (oracle/pcv_oracle.c) is pinned against, and the `--impl reference`
// CPU arm of bench.py. Never linked into the product.
#include <chrono>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "../include/pcvg.h"
#include "pcv/adapt.hpp"
#include "pcv/models/registry.hpp"
#include "pcv/report_io.hpp"
#include "pcv/config.hpp"
#include "pcv/diagnostics.hpp"
#include "pcv/accum.hpp"
#include "pcv/engine.hpp"
#include "pcv/errors.hpp"
#include "pcv/folds.hpp"
#include "pcv/hmc.hpp"
#include "pcv/models/grouped_regression.hpp"
#include "pcv/models/radon.hpp"
#include "pcv/models/rat_growth.hpp"
#include "pcv/models/seasonal_ar.hpp"
#include "pcv/rng.hpp"
#include "ref_plugins.hpp"

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PCVG_OK;
  } catch (const pcv::invalid_input& e) {
    return fail(PCVG_INVALID_INPUT, e.what());
  } catch (const pcv::numeric_fault& e) {
    return fail(PCVG_NUMERIC_FAULT, e.what());
  } catch (const pcv::adaptation_failure& e) {
    return fail(PCVG_ADAPTATION_FAILURE, e.what());
  } catch (const pcv::undefined_diagnostic& e) {
    return fail(PCVG_UNDEFINED_DIAGNOSTIC, e.what());
  } catch (const pcv::unsupported_score& e) {
    return fail(PCVG_UNSUPPORTED_SCORE, e.what());
  } catch (const std::exception& e) {
    return fail(PCVG_INVALID_INPUT, e.what());
  }
}

pcv::Dataset to_dataset(const pcvg_dataset* d) {
  pcv::Dataset out;
  const long n = static_cast<long>(d->n_obs);
  out.n_cov = d->n_cov;
  out.y.assign(d->y, d->y + n);
  if (d->n_cov > 0) out.x.assign(d->x, d->x + n * d->n_cov);
  if (d->group_id) out.group_id.assign(d->group_id, d->group_id + n);
  if (d->time_index) out.time_index.assign(d->time_index, d->time_index + n);
  return out;
}

struct RefModel {
  std::unique_ptr<pcv::Model> model;
};

}  // namespace

extern "C" {

const char* pcvref_last_error() { return g_err.c_str(); }

uint64_t pcvref_stream_key(uint64_t kind, uint64_t a, uint64_t b, uint64_t c) {
  return pcv::stream_key(static_cast<pcv::StreamKind>(kind), a, b, c);
}

int pcvref_rng_sequence(uint64_t seed, uint64_t stream, int32_t do_skip, uint64_t skip_block,
                        const char* ops, const uint64_t* arg, int64_t n, double* out) {
  return guarded([&] {
    pcv::CounterRng rng(seed, stream);
    if (do_skip) rng.skip_to(skip_block);
    for (int64_t i = 0; i < n; ++i) {
      switch (ops[i]) {
        case 'u': out[i] = rng.uniform(); break;
        case 'n': out[i] = rng.normal(); break;
        case '4': out[i] = static_cast<double>(rng.next_u32()); break;
        case 'b': out[i] = static_cast<double>(rng.below(arg[i])); break;
        default: throw pcv::invalid_input("bad rng op");
      }
    }
  });
}

int pcvref_make_kfold(int64_t n, int32_t K, uint64_t seed, int32_t* out) {
  return guarded([&] {
    pcv::Dataset d;
    d.y.assign(n, 0.0);
    const auto f = pcv::make_kfold_scheme(d, K, seed);
    std::memcpy(out, f.test_index.data(), sizeof(int32_t) * n);
  });
}

int pcvref_make_time_blocks(const pcvg_dataset* ds, int32_t K, int32_t* out) {
  return guarded([&] {
    const auto f = pcv::make_time_block_scheme(to_dataset(ds), K);
    std::memcpy(out, f.test_index.data(), sizeof(int32_t) * ds->n_obs);
  });
}

int pcvref_make_logo(const pcvg_dataset* ds, int32_t* out, int32_t* K) {
  return guarded([&] {
    const auto f = pcv::make_logo_scheme(to_dataset(ds));
    std::memcpy(out, f.test_index.data(), sizeof(int32_t) * ds->n_obs);
    *K = f.K;
  });
}

int pcvref_simulate_grouped(int32_t J, int32_t Nj, int32_t P, double min_beta, uint64_t seed,
                            double* y, double* x, int32_t* g) {
  return guarded([&] {
    pcv::GroupedSimOptions o;
    o.groups = J;
    o.per_group = Nj;
    o.covariates = P;
    o.min_omitted_beta = min_beta;
    const auto r = pcv::simulate_grouped_regression(o, seed);
    std::memcpy(y, r.data.y.data(), sizeof(double) * r.data.y.size());
    std::memcpy(x, r.data.x.data(), sizeof(double) * r.data.x.size());
    std::memcpy(g, r.data.group_id.data(), sizeof(int32_t) * r.data.group_id.size());
  });
}

int pcvref_simulate_rat(int32_t subjects, uint64_t seed, double* y, double* x, int32_t* g) {
  return guarded([&] {
    const auto r = pcv::simulate_rat_growth(subjects, seed);
    std::memcpy(y, r.data.y.data(), sizeof(double) * r.data.y.size());
    std::memcpy(x, r.data.x.data(), sizeof(double) * r.data.x.size());
    for (size_t i = 0; i < r.data.group_id.size(); ++i) g[i] = r.data.group_id[i];
  });
}

int pcvref_simulate_radon(int32_t houses, int32_t counties, uint64_t seed, double* y, double* x,
                          int32_t* g) {
  return guarded([&] {
    const auto r = pcv::simulate_radon_style(houses, counties, seed);
    std::memcpy(y, r.data.y.data(), sizeof(double) * r.data.y.size());
    std::memcpy(x, r.data.x.data(), sizeof(double) * r.data.x.size());
    std::memcpy(g, r.data.group_id.data(), sizeof(int32_t) * r.data.group_id.size());
  });
}

// cfg2 logistic simulator (the logistic family is a plugin, ref_plugins.hpp): the same draw order
// as the product's pcvg_simulate_logistic on the reference's own CounterRng, so the reference arm
// of bench.py builds its inputs without the product library.
int pcvref_simulate_logistic(int64_t n, int32_t P, uint64_t seed, double* y, double* x) {
  return guarded([&] {
    if (n < 2 || P < 1) throw pcv::invalid_input("logistic simulator needs n >= 2, P >= 1");
    pcv::CounterRng rng(seed, pcv::stream_key(pcv::StreamKind::Simulate, 5));
    std::vector<double> beta(P + 1);
    for (double& b : beta) b = rng.normal();
    const double scale = 1.0 / std::sqrt(static_cast<double>(P));
    for (int64_t i = 0; i < n; ++i) {
      double eta = beta[0];
      for (int32_t j = 0; j < P; ++j) {
        x[i * P + j] = rng.normal() * scale;
        eta += x[i * P + j] * beta[1 + j];
      }
      y[i] = rng.uniform() < 1.0 / (1.0 + std::exp(-eta)) ? 1.0 : 0.0;
    }
  });
}

int pcvref_simulate_seasonal(int64_t months, int32_t p, int32_t q, double rho, double amp,
                             double sigma, uint64_t seed, double* y, double* x, int64_t* t) {
  return guarded([&] {
    pcv::SeasonalSimOptions o;
    o.months = months;
    o.ar_order = p;
    o.dummies = q;
    o.rho = rho;
    o.seasonal_amp = amp;
    o.sigma = sigma;
    const auto r = pcv::simulate_seasonal_ar(o, seed);
    std::memcpy(y, r.data.y.data(), sizeof(double) * r.data.y.size());
    std::memcpy(x, r.data.x.data(), sizeof(double) * r.data.x.size());
    for (size_t i = 0; i < r.data.time_index.size(); ++i) t[i] = r.data.time_index[i];
  });
}

// Builds a reference Model (or an oracle plugin on the reference API) from a descriptor.
void* pcvref_model_create(const pcvg_dataset* ds, const pcvg_folds* fs,
                          const pcvg_model_spec* spec, const char* name) {
  RefModel* out = nullptr;
  const int rc = guarded([&] {
    pcv::Dataset d = to_dataset(ds);
    auto rm = std::make_unique<RefModel>();
    const std::string nm = name ? name : "M";
    if (fs->intervals) {
      if (spec->family != PCVG_FAMILY_SEASONAL_AR)
        throw pcv::invalid_input("hv-block folds are only wired for seasonal-ar");
      std::vector<pcvoracle::HvFold> hv(fs->K);
      for (int k = 0; k < fs->K; ++k)
        hv[k] = {fs->intervals[4 * k], fs->intervals[4 * k + 1], fs->intervals[4 * k + 2],
                 fs->intervals[4 * k + 3]};
      rm->model = std::make_unique<pcvoracle::HvSeasonalARModel>(
          nm, d, std::move(hv), spec->ar_order, spec->dummies,
          spec->rho_transform == PCVG_RHO_SYMMETRIC ? pcv::RhoTransform::Symmetric
                                                    : pcv::RhoTransform::HalfOpen);
    } else {
      pcv::FoldAssignment f;
      f.K = fs->K;
      f.test_index.assign(fs->test_index, fs->test_index + ds->n_obs);
      switch (spec->family) {
        case PCVG_FAMILY_GROUPED: {
          std::vector<int> mask;
          if (spec->covariate_mask) mask.assign(spec->covariate_mask, spec->covariate_mask + ds->n_cov);
          rm->model = std::make_unique<pcv::GroupedRegressionModel>(nm, std::move(d), std::move(f), mask);
          break;
        }
        case PCVG_FAMILY_RADON:
          rm->model = std::make_unique<pcv::RadonStyleModel>(nm, std::move(d), std::move(f),
                                                             spec->include_floor != 0);
          break;
        case PCVG_FAMILY_SEASONAL_AR:
          rm->model = std::make_unique<pcv::SeasonalARModel>(
              nm, std::move(d), std::move(f), spec->ar_order, spec->dummies,
              spec->rho_transform == PCVG_RHO_SYMMETRIC ? pcv::RhoTransform::Symmetric
                                                        : pcv::RhoTransform::HalfOpen);
          break;
        case PCVG_FAMILY_LOGISTIC:
          rm->model = std::make_unique<pcvoracle::LogisticModel>(nm, std::move(d), std::move(f));
          break;
        case PCVG_FAMILY_RAT_GROWTH:
          rm->model = std::make_unique<pcv::RatGrowthModel>(nm, std::move(d), std::move(f),
                                                            spec->per_subject_slope != 0);
          break;
        default:
          throw pcv::invalid_input("family not wired in the reference shim");
      }
    }
    out = rm.release();
  });
  return rc == PCVG_OK ? out : nullptr;
}

void pcvref_model_destroy(void* h) { delete static_cast<RefModel*>(h); }

static const pcv::Model& M(void* h) { return *static_cast<RefModel*>(h)->model; }

int32_t pcvref_model_dim(void* h) { return M(h).dim(); }
int64_t pcvref_test_size(void* h, int32_t fold) { return M(h).test_size(fold); }

double pcvref_log_joint(void* h, const double* theta, int32_t fold) {
  return M(h).log_joint({theta, static_cast<size_t>(M(h).dim())}, fold);
}
void pcvref_grad(void* h, const double* theta, int32_t fold, double* grad) {
  const size_t d = M(h).dim();
  M(h).grad_log_joint({theta, d}, fold, {grad, d});
}
double pcvref_log_pred(void* h, const double* theta, int32_t fold) {
  return M(h).log_pred({theta, static_cast<size_t>(M(h).dim())}, fold);
}
double pcvref_log_lik_test(void* h, const double* theta, int32_t fold) {
  return M(h).log_lik_test({theta, static_cast<size_t>(M(h).dim())}, fold);
}
// Model::pred_derivs / pred_sample (model.hpp:54-66); returns 0, or 1 when unsupported.
int pcvref_pred_derivs(void* h, const double* theta, int32_t fold, double* d1, double* d2) {
  if (!M(h).supports_pred_derivs()) return 1;
  const size_t n = M(h).test_size(fold);
  M(h).pred_derivs({theta, static_cast<size_t>(M(h).dim())}, fold, {d1, n}, {d2, n});
  return 0;
}
int pcvref_pred_sample(void* h, const double* theta, int32_t fold, uint64_t seed, uint64_t stream,
                       int32_t times, double* out) {
  if (!M(h).supports_pred_sample()) return 1;
  const size_t n = M(h).test_size(fold);
  pcv::CounterRng rng(seed, stream);
  for (int32_t r = 0; r < times; ++r)
    M(h).pred_sample({theta, static_cast<size_t>(M(h).dim())}, fold, rng, {out + r * n, n});
  return 0;
}
void pcvref_initial_draw(void* h, uint64_t seed, uint64_t stream, double* out) {
  pcv::CounterRng rng(seed, stream);
  const auto v = M(h).initial_draw(rng);
  std::memcpy(out, v.data(), sizeof(double) * v.size());
}

int32_t pcvref_leapfrog(void* h, int32_t fold, double step, int32_t n_lf, const double* inv_mass,
                        double* q, double* p) {
  const size_t d = M(h).dim();
  std::vector<double> grad(d);
  return pcv::leapfrog({q, d}, {p, d}, M(h), fold, step, n_lf, {inv_mass, d}, grad) ? 1 : 0;
}

// n consecutive reference hmc_step calls on stream CounterRng(seed, stream).
int pcvref_hmc_chain(void* h, int32_t fold, double step, int32_t n_lf, const double* inv_mass,
                     uint64_t seed, uint64_t stream, const double* theta0, int64_t n_steps,
                     double* traj, int32_t* divergent, int32_t* accepted, double* delta_h) {
  return guarded([&] {
    const size_t d = M(h).dim();
    pcv::KernelParams kp{step, n_lf, std::vector<double>(inv_mass, inv_mass + d)};
    pcv::ChainState st{std::vector<double>(theta0, theta0 + d), pcv::CounterRng(seed, stream), 0};
    pcv::HmcWorkspace ws;
    for (int64_t s = 0; s < n_steps; ++s) {
      const auto info = pcv::hmc_step(st, M(h), fold, kp, ws);
      std::memcpy(traj + s * d, st.position.data(), sizeof(double) * d);
      if (divergent) divergent[s] = info.divergent;
      if (accepted) accepted[s] = info.accepted;
      if (delta_h) delta_h[s] = info.delta_h;
    }
  });
}

int pcvref_adapt(void* h, int32_t chains, int64_t warmup, int64_t draws, int32_t n_lf,
                 double target, double init_step, uint64_t seed, int32_t model_id,
                 double* step_out, double* inv_mass_out, double* bank_out, double* mean_accept,
                 int64_t* divergences) {
  return guarded([&] {
    pcv::AdaptConfig ac;
    ac.chains = chains;
    ac.warmup = warmup;
    ac.draws = draws;
    ac.n_leapfrog = n_lf;
    ac.target_accept = target;
    ac.init_step_size = init_step;
    const auto fit = pcv::adapt_full_data(M(h), ac, seed, model_id);
    *step_out = fit.kparams.step_size;
    const size_t d = M(h).dim();
    std::memcpy(inv_mass_out, fit.kparams.inv_mass_diag.data(), sizeof(double) * d);
    for (size_t r = 0; r < fit.draws.size(); ++r)
      std::memcpy(bank_out + r * d, fit.draws[r].data(), sizeof(double) * d);
    if (mean_accept) *mean_accept = fit.mean_accept;
    if (divergences) *divergences = fit.divergences;
  });
}

// Test oracle: adapt_full_data (adapt.cpp:96-185) restated over the reference's public pieces
// (hmc_step, DualAveraging, WelfordDiag) with per-iteration traces, to localise differences
// between the device adaptation and the reference. Returns the initial step size.
int pcvref_adapt_trace(void* h, int32_t chains, int64_t warmup, int32_t n_lf, double target,
                       uint64_t seed, int32_t model_id, double* init_step, double* step_trace,
                       double* ap_trace, double* inv_mass_out, double* pos_out) {
  return guarded([&] {
    const pcv::Model& model = M(h);
    const int d = model.dim(), sentinel = model.fold_count(), l = chains;
    std::vector<pcv::ChainState> cs;
    for (int c = 0; c < l; ++c) {
      pcv::CounterRng rng(seed, pcv::stream_key(pcv::StreamKind::FullData,
                                                static_cast<std::uint64_t>(model_id),
                                                static_cast<std::uint64_t>(c)));
      cs.push_back(pcv::ChainState{model.initial_draw(rng), rng, 0});
    }
    if (pos_out)
      for (int c = 0; c < l; ++c) std::memcpy(pos_out + c * d, cs[c].position.data(), sizeof(double) * d);
    pcv::KernelParams kp;
    kp.n_leapfrog = n_lf;
    kp.inv_mass_diag.assign(d, 1.0);
    pcv::HmcWorkspace ws;
    auto probe = [&](double e) {  // find_initial_step, adapt.cpp:17-43
      pcv::ChainState ps{cs[0].position,
                         pcv::CounterRng(seed, pcv::stream_key(pcv::StreamKind::StepInit,
                                                               static_cast<std::uint64_t>(model_id))),
                         0};
      pcv::KernelParams k1{e, 1, kp.inv_mass_diag};
      const auto info = pcv::hmc_step(ps, model, sentinel, k1, ws);
      return info.divergent ? 0.0 : info.accept_prob;
    };
    double eps = 1.0;
    const bool go_up = probe(eps) > 0.5;
    bool done = false;
    for (int i = 0; i < 50 && !done; ++i) {
      if (go_up) {
        eps *= 2.0;
        if (probe(eps) <= 0.5) { eps /= 2.0; done = true; }
      } else {
        eps *= 0.5;
        if (probe(eps) > 0.5) done = true;
      }
    }
    kp.step_size = done ? eps : (go_up ? eps : 1e-8);
    *init_step = kp.step_size;
    pcv::DualAveraging da;
    da.target = target;
    da.restart(kp.step_size);
    const long w_total = warmup;
    const long w_init = std::min<long>(75, std::max<long>(1, w_total * 15 / 100));
    const long w_final = std::min<long>(50, std::max<long>(1, w_total / 10));
    long window = 25;
    long window_end = std::min(w_total - w_final, w_init + window);
    pcv::WelfordDiag acc(d);
    for (long iter = 0; iter < w_total; ++iter) {
      kp.step_size = da.current();
      step_trace[iter] = kp.step_size;
      double ap = 0.0;
      for (auto& ch : cs) {
        const auto info = pcv::hmc_step(ch, model, sentinel, kp, ws);
        ap += info.divergent ? 0.0 : info.accept_prob;
      }
      ap /= l;
      ap_trace[iter] = ap;
      da.update(ap);
      const bool in_slow = iter >= w_init && iter < w_total - w_final;
      if (in_slow)
        for (const auto& ch : cs) acc.add(ch.position);
      if (in_slow && iter + 1 == window_end) {
        if (acc.count() >= 2) {
          const auto var = acc.variance();
          const double n = static_cast<double>(acc.count());
          for (int i = 0; i < d; ++i)
            kp.inv_mass_diag[i] = std::max(var[i] * (n / (n + 5.0)) + 1e-3 * (5.0 / (n + 5.0)), 1e-10);
        }
        acc = pcv::WelfordDiag(d);
        da.restart(da.current());
        window *= 2;
        long next_end = window_end + window;
        if (next_end + 2 * window > w_total - w_final) next_end = w_total - w_final;
        window_end = next_end;
      }
    }
    std::memcpy(inv_mass_out, kp.inv_mass_diag.data(), sizeof(double) * d);
  });
}

// The reference's own file writers/readers (registry.cpp:98-165, report_io.cpp), for the CLI
// format tests: run_simulator with "key=value;..." arguments; read_full_data_fit.
int pcvref_run_simulator(const char* family, const char* args, uint64_t seed, const char* out_dir) {
  return guarded([&] {
    pcv::ConfigMap a;
    std::string s(args ? args : "");
    size_t pos = 0;
    while (pos < s.size()) {
      size_t end = s.find(';', pos);
      if (end == std::string::npos) end = s.size();
      const std::string kv = s.substr(pos, end - pos);
      const size_t eq = kv.find('=');
      if (eq != std::string::npos) a.set(kv.substr(0, eq), kv.substr(eq + 1));
      pos = end + 1;
    }
    pcv::run_simulator(family, a, seed, out_dir);
  });
}

int pcvref_read_fit(const char* dir, const char* stem, int64_t* rows, int64_t* cols, double* step,
                    double* first_row) {
  return guarded([&] {
    const auto fit = pcv::read_full_data_fit(dir, stem);
    *rows = static_cast<int64_t>(fit.draws.size());
    *cols = fit.draws.empty() ? 0 : static_cast<int64_t>(fit.draws[0].size());
    *step = fit.kparams.step_size;
    if (first_row && !fit.draws.empty())
      std::memcpy(first_row, fit.draws[0].data(), sizeof(double) * fit.draws[0].size());
  });
}

// Reference run_pcv written with the reference writers (report.json, progressive.csv, benchmark.csv).
int pcvref_run_pcv_files(int32_t n_models, void** models, const int32_t* model_ids,
                         const pcvg_kernel* kernels, const double* const* banks, const int64_t* bank_rows,
                         const pcvg_run_config* c, int32_t threads, const char* out_dir) {
  return guarded([&] {
    pcv::RunConfig cfg;
    cfg.chains = c->chains;
    cfg.iters = c->iters;
    cfg.warmup = c->warmup;
    cfg.batch_size = c->batch_size;
    cfg.blocks = c->blocks;
    cfg.bench_draws = c->bench_draws;
    cfg.bench_quantile = c->bench_quantile;
    cfg.seed = c->seed;
    cfg.score = static_cast<pcv::ScoreKind>(c->score);
    cfg.checkpoint_every = c->checkpoint_every;
    cfg.thread_budget = threads;
    std::vector<pcv::FullDataFit> fits(n_models);
    std::vector<pcv::ModelInput> inputs;
    for (int m = 0; m < n_models; ++m) {
      const size_t d = M(models[m]).dim();
      fits[m].kparams.step_size = kernels[m].step_size;
      fits[m].kparams.n_leapfrog = kernels[m].n_leapfrog;
      fits[m].kparams.inv_mass_diag.assign(kernels[m].inv_mass_diag, kernels[m].inv_mass_diag + d);
      for (int64_t r = 0; r < bank_rows[m]; ++r)
        fits[m].draws.emplace_back(banks[m] + r * d, banks[m] + (r + 1) * d);
      inputs.push_back({&M(models[m]), &fits[m], model_ids[m]});
    }
    const pcv::PcvReport r = pcv::run_pcv(inputs, cfg);
    const std::string dir(out_dir);
    pcv::write_report_json(dir + "/report.json", r);
    pcv::write_progressive_csv(dir + "/progressive.csv", r);
    pcv::write_benchmark_csv(dir + "/benchmark.csv", r);
  });
}

int pcvref_run_pcv(int32_t n_models, void** models, const int32_t* model_ids,
                   const pcvg_kernel* kernels, const double* const* banks,
                   const int64_t* bank_rows, const pcvg_run_config* c, int32_t threads,
                   pcvg_report* rep) {
  return guarded([&] {
    pcv::RunConfig cfg;
    cfg.chains = c->chains;
    cfg.iters = c->iters;
    cfg.warmup = c->warmup;
    cfg.batch_size = c->batch_size;
    cfg.blocks = c->blocks;
    cfg.bench_draws = c->bench_draws;
    cfg.bench_quantile = c->bench_quantile;
    cfg.seed = c->seed;
    cfg.score = static_cast<pcv::ScoreKind>(c->score);
    cfg.checkpoint_every = c->checkpoint_every;
    cfg.thread_budget = threads;
    cfg.shared_streams = c->shared_streams != 0;
    std::vector<pcv::FullDataFit> fits(n_models);
    std::vector<pcv::ModelInput> inputs;
    for (int m = 0; m < n_models; ++m) {
      const size_t d = M(models[m]).dim();
      fits[m].kparams.step_size = kernels[m].step_size;
      fits[m].kparams.n_leapfrog = kernels[m].n_leapfrog;
      fits[m].kparams.inv_mass_diag.assign(kernels[m].inv_mass_diag,
                                           kernels[m].inv_mass_diag + d);
      for (int64_t r = 0; r < bank_rows[m]; ++r)
        fits[m].draws.emplace_back(banks[m] + r * d, banks[m] + (r + 1) * d);
      inputs.push_back({&M(models[m]), &fits[m], model_ids[m]});
    }
    const pcv::PcvReport r = pcv::run_pcv(inputs, cfg);
    const int K = r.folds, L = r.chains;
    for (int m = 0; m < n_models; ++m) {
      const auto& mr = r.models[m];
      for (int k = 0; k < K; ++k) {
        const auto& fs = mr.folds[k];
        const size_t i = static_cast<size_t>(m) * K + k;
        rep->folds.estimate[i] = fs.estimate;
        rep->folds.log_f_hat[i] = fs.log_f_hat;
        rep->folds.mc_contribution[i] = fs.mc_contribution;
        if (rep->folds.naive_contribution) rep->folds.naive_contribution[i] = NAN;
        rep->folds.ess[i] = fs.ess;
        rep->folds.rhat[i] = fs.rhat;
        rep->folds.batches[i] = fs.batches;
        rep->folds.fault[i] = fs.fault;
        rep->folds.failed[i] = fs.failed;
        if (rep->folds.dss_ridged) rep->folds.dss_ridged[i] = fs.dss_ridged;
        for (int ch = 0; ch < L; ++ch)
          rep->divergences[(i)*L + ch] = mr.divergences[k][ch];
      }
      rep->score_total[m] = mr.score_total;
      rep->numeric_faults[m] = mr.numeric_faults;
      rep->rhat_excluded[m] = mr.rhat_excluded;
    }
    for (int k = 0; k < K; ++k) rep->delta_k[k] = r.delta_k[k];
    rep->n_checkpoints = static_cast<int32_t>(r.snapshots.size());
    for (size_t s = 0; s < r.snapshots.size(); ++s) {
      const auto& sn = r.snapshots[s];
      double* o = rep->snapshots + 7 * s;
      o[0] = static_cast<double>(sn.iteration);
      o[1] = sn.delta_hat;
      o[2] = sn.mcse;
      o[3] = sn.epistemic_se;
      o[4] = sn.prob_a_better;
      o[5] = sn.ess;
      o[6] = sn.rhat_max;
    }
    rep->benchmark_count = static_cast<int32_t>(r.benchmark.values.size());
    for (size_t b = 0; b < r.benchmark.values.size(); ++b) rep->benchmark[b] = r.benchmark.values[b];
    rep->delta_hat = r.delta_hat;
    rep->mcse = r.mcse;
    rep->sigma2_delta = r.sigma2_delta;
    rep->epistemic_se = r.epistemic_se;
    rep->prob_a_better = r.prob_a_better;
    rep->ess_overall = r.ess_overall;
    rep->rhat_max = r.rhat_max;
    rep->dropped_batch_draws = r.dropped_batch_draws;
    rep->verdict_pass = r.verdict.pass;
    rep->verdict_quantile = r.verdict.quantile;
    rep->verdict_quantile_value = r.verdict.quantile_value;
    rep->verdict_observed = r.verdict.observed;
    rep->iters_run = r.iters;
  });
}

// The reference's shuffle-benchmark acceptance harness (acceptance.cpp:259-325, criteria C6/C7) run
// on the reference library: K = 10 folds x L = 4 autocorrelated score chains of n = 1000 draws
// (rho = 0.3, fold locations 2 N(0,1), overdispersed start), optionally one corrupted chain of
// fold 2 (kind 1 = stuck at its start, kind 2 = shifted by +5), fed through ScoreAccum(b = 50,
// D = 5, n, mu_k); returns the observed R-hat max, the 0.99 nearest-rank benchmark quantile of R
// replicates and the verdict. tests/golden/make_acceptance.py stores them for the device runs.
int pcvref_corrupted_run(int32_t seed, int32_t kind, int32_t bench_draws, double* observed,
                         double* quantile_value, int32_t* pass) {
  return guarded([&] {
    const int k_folds = 10, l = 4, d_blocks = 5, b = 50;
    const long n = 1000;
    const int bad_fold = 2, bad_chain = 0;
    const double rho = 0.3;
    const std::uint64_t run_seed = 7000 + static_cast<std::uint64_t>(seed);
    std::vector<std::vector<pcv::ScoreAccum>> acc(k_folds);
    for (int k = 0; k < k_folds; ++k) {
      pcv::CounterRng fold_rng(run_seed, pcv::stream_key(pcv::StreamKind::Simulate, static_cast<std::uint64_t>(k)));
      const double mu_k = 2.0 * fold_rng.normal();
      for (int c = 0; c < l; ++c) {
        pcv::CounterRng rng(run_seed, pcv::stream_key(pcv::StreamKind::ChainSampling, 0, static_cast<std::uint64_t>(k),
                                                      static_cast<std::uint64_t>(c)));
        const bool corrupt = kind != 0 && k == bad_fold && c == bad_chain;
        const double start = mu_k + 3.0;
        double state = start - mu_k;
        const double innov = std::sqrt(1.0 - rho * rho);
        pcv::ScoreAccum a(b, d_blocks, n, mu_k);
        for (long i = 0; i < n; ++i) {
          state = rho * state + innov * rng.normal();
          double v = (corrupt && kind == 1) ? start : mu_k + state;
          if (corrupt && kind == 2) v += 5.0;
          a.observe(v, i);
        }
        acc[k].push_back(std::move(a));
      }
    }
    std::vector<double> rhats;
    std::vector<pcv::FoldBlockSums> blocks;
    for (int k = 0; k < k_folds; ++k) {
      const auto st = pcv::rhat_from_blocks(acc[k], n);
      rhats.push_back(st ? st->rhat : std::numeric_limits<double>::quiet_NaN());
      blocks.push_back(pcv::gather_block_sums(acc[k], n));
    }
    const double obs = pcv::rhat_max(rhats);
    const auto bench = pcv::shuffle_benchmark(blocks, bench_draws, run_seed);
    const auto v = pcv::benchmark_verdict(obs, bench, 0.99);
    *observed = v.observed;
    *quantile_value = v.quantile_value;
    *pass = v.pass ? 1 : 0;
  });
}

}  // extern "C"

extern "C" {

// Times the reference's own Step 2-3 task loop (engine.cpp:296-381: warm start, warmup_discard,
// then hmc_step + log_pred + ScoreAccum::observe per iteration) on a bounded sample of folds with
// the reference thread pool (parallel_for, engine.cpp:32-61). Used by bench.py's CPU arms.
int pcvref_time_tasks(void* h, int32_t n_folds, const int32_t* folds, int32_t L, int64_t warmup,
                      int64_t iters, uint64_t seed, int32_t model_id, const pcvg_kernel* kern,
                      const double* bank, int64_t bank_rows, int32_t threads, double* sampling_s,
                      double* warmup_s, double* checksum) {
  return guarded([&] {
    const pcv::Model& model = M(h);
    const size_t d = model.dim();
    pcv::KernelParams kp{kern->step_size, kern->n_leapfrog,
                         std::vector<double>(kern->inv_mass_diag, kern->inv_mass_diag + d)};
    struct Task {
      pcv::ChainState st{{}, pcv::CounterRng(), 0};
      pcv::WarmupStats warm;
      pcv::ScoreAccum acc;
      int fold = 0, chain = 0;
    };
    const long ntask = static_cast<long>(n_folds) * L;
    std::vector<Task> tasks(ntask);
    for (long i = 0; i < ntask; ++i) {
      tasks[i].fold = folds[i / L];
      tasks[i].chain = static_cast<int>(i % L);
    }
    auto t0 = std::chrono::steady_clock::now();
    pcv::parallel_for(ntask, threads, [&](long i) {
      Task& t = tasks[i];
      pcv::CounterRng init(seed, pcv::stream_key(pcv::StreamKind::ChainInit, model_id, t.fold, t.chain));
      const uint64_t row = init.below(static_cast<uint64_t>(bank_rows));
      t.st.position.assign(bank + row * d, bank + (row + 1) * d);
      t.st.rng = pcv::CounterRng(seed, pcv::stream_key(pcv::StreamKind::ChainSampling, model_id, t.fold, t.chain));
      pcv::HmcWorkspace ws;
      t.warm = pcv::warmup_discard(t.st, model, t.fold, kp, warmup, pcv::ScoreKind::LogS, ws);
    });
    auto t1 = std::chrono::steady_clock::now();
    const int b = static_cast<int>(std::min<int64_t>(50, iters));
    pcv::parallel_for(ntask, threads, [&](long i) {
      Task& t = tasks[i];
      const double c = warmup > 0 ? t.warm.logpred_sum / (static_cast<double>(L) * warmup) : 0.0;
      t.acc = pcv::ScoreAccum(b, 5, iters, c);
      pcv::HmcWorkspace ws;
      for (int64_t it = 0; it < iters; ++it) {
        pcv::hmc_step(t.st, model, t.fold, kp, ws);
        t.acc.observe(model.log_pred(t.st.position, t.fold), it);
      }
    });
    auto t2 = std::chrono::steady_clock::now();
    *warmup_s = std::chrono::duration<double>(t1 - t0).count();
    *sampling_s = std::chrono::duration<double>(t2 - t1).count();
    double cs = 0.0;
    for (const auto& t : tasks) cs += t.acc.raw.u_x;
    *checksum = cs;
  });
}

}  // extern "C"
