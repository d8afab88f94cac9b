/*
 * pcvg.h - C ABI of the B200-native parallel-CV (PCV) sampler (libpcvg.so).
 *
 * Drop-in boundary for Steps 2-3 of the reference engine, i.e. the region
 *   pcv::run_pcv  /root/reference/proj/src/engine.cpp:295-381
 * (warm start + fold warm-up + sampling into online accumulators), plus the Step-4
 * reductions it feeds (engine.cpp:117-253, 385-480). A GPU cannot call a host virtual
 * per observation, so the swap point sits one level above `class pcv::Model`
 * (include/pcv/model.hpp:24-78): the caller hands over a *model descriptor*
 * (family + dataset + fold scheme + family options) instead of a `Model*`.
 *
 * Conventions (all mirror the reference):
 *  - every function returns a pcvg_status; no exception crosses the ABI;
 *    the status codes map the reference error taxonomy (include/pcv/errors.hpp:9-37);
 *  - buffers are caller-owned plain pointers + sizes (the reference's std::span);
 *  - fold id K is the full-data sentinel (model.hpp:17-20);
 *  - task order is (m*K + k)*L + c (engine.cpp:289, 747-755);
 *  - a context is single-caller (the reference's coordinator thread, engine.hpp:5-6).
 * There are no torch types here: plain C, usable from C, C++, ctypes, cgo, JNI.
 */
#ifndef PCVG_H
#define PCVG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCVG_ABI_VERSION 3

typedef enum {
  PCVG_OK = 0,
  PCVG_INVALID_INPUT = 1,         /* pcv::invalid_input       errors.hpp:15-17 */
  PCVG_NUMERIC_FAULT = 2,         /* pcv::numeric_fault       errors.hpp:19-21 */
  PCVG_ADAPTATION_FAILURE = 3,    /* pcv::adaptation_failure  errors.hpp:23-28 */
  PCVG_UNDEFINED_DIAGNOSTIC = 4,  /* pcv::undefined_diagnostic errors.hpp:30-32 */
  PCVG_UNSUPPORTED_SCORE = 5,     /* pcv::unsupported_score   errors.hpp:34-36 */
  PCVG_CUDA_ERROR = 6,            /* device failure (new) */
  PCVG_COMM_ERROR = 7             /* collective failure (new) */
} pcvg_status;

/* Model families (the reference's src/models/*.cpp, plus the new logistic family). */
typedef enum {
  PCVG_FAMILY_GROUPED = 0,     /* GroupedRegressionModel  grouped_regression.hpp:23-77 */
  PCVG_FAMILY_RADON = 1,       /* RadonStyleModel         radon.hpp:18-64 */
  PCVG_FAMILY_SEASONAL_AR = 2, /* SeasonalARModel         seasonal_ar.hpp:22-61 */
  PCVG_FAMILY_LOGISTIC = 3,    /* new: Bernoulli-logit regression (BASELINE configs[1]) */
  PCVG_FAMILY_RAT_GROWTH = 4   /* RatGrowthModel (rat_growth.hpp:20-63); per_subject_slope = M_A */
} pcvg_family;

typedef enum { PCVG_SCORE_LOGS = 0, PCVG_SCORE_HS = 1, PCVG_SCORE_DSS = 2 } pcvg_score; /* model.hpp:12 */
typedef enum { PCVG_RHO_HALF_OPEN = 0, PCVG_RHO_SYMMETRIC = 1 } pcvg_rho_transform;   /* seasonal_ar.hpp:20 */

/* Stream purpose tags, rng.hpp:25-33. */
typedef enum {
  PCVG_STREAM_CHAIN_SAMPLING = 1, PCVG_STREAM_CHAIN_INIT = 2, PCVG_STREAM_FULL_DATA = 3,
  PCVG_STREAM_SIMULATE = 4, PCVG_STREAM_KFOLD = 5, PCVG_STREAM_BENCHMARK = 6,
  PCVG_STREAM_STEP_INIT = 7
} pcvg_stream_kind;

/* Column store, pcv::Dataset (dataset.hpp:11-25). */
typedef struct {
  int64_t n_obs;
  int32_t n_cov;
  const double* y;            /* [n_obs] */
  const double* x;            /* [n_obs * n_cov], row-major */
  const int32_t* group_id;    /* [n_obs], contiguous 0..J-1, or NULL */
  const int64_t* time_index;  /* [n_obs] or NULL */
} pcvg_dataset;

/* Fold scheme. Either a partition pcv::FoldAssignment (folds.hpp:10-20: test_index[n_obs]
 * in 0..K-1) or, for hv-block CV (new; SPEC.md:114 left it unimplemented), K interval
 * folds over the time rank: intervals[4k..4k+3] = {test_lo, test_hi, ex_lo, ex_hi}; fold k
 * scores ranks [test_lo, test_hi) and trains on ranks outside [ex_lo, ex_hi). */
typedef struct {
  int32_t K;
  const int32_t* test_index;  /* partition, or NULL */
  const int64_t* intervals;   /* hv-block, or NULL */
} pcvg_folds;

/* Family options (registry.cpp:55-91). */
typedef struct {
  int32_t family;                 /* pcvg_family */
  const int32_t* covariate_mask;  /* grouped: [n_cov] or NULL = all on (grouped_regression.cpp:123) */
  int32_t include_floor;          /* radon (radon.hpp:20-23) */
  int32_t ar_order;               /* seasonal: p */
  int32_t dummies;                /* seasonal: q */
  int32_t rho_transform;          /* seasonal: pcvg_rho_transform */
  int32_t per_subject_slope;      /* rat growth */
} pcvg_model_spec;

/* pcv::KernelParams (hmc.hpp:14-18). */
typedef struct {
  double step_size;
  int32_t n_leapfrog;
  const double* inv_mass_diag;  /* [dim] */
} pcvg_kernel;

/* pcv::RunConfig (engine.hpp:21-45), sampling part, plus sharding / early stop. */
typedef struct {
  int32_t chains;          /* L >= 2 */
  int64_t iters;           /* N */
  int64_t warmup;          /* N_wu */
  int32_t batch_size;      /* b; 0 = floor(sqrt(N L)) (engine.cpp:5-9) */
  int32_t blocks;          /* D */
  int32_t bench_draws;     /* R */
  double bench_quantile;   /* 0.99 */
  uint64_t seed;
  int32_t score;           /* pcvg_score */
  int64_t checkpoint_every;
  int32_t shared_streams;
  int32_t fold_begin;      /* shard [fold_begin, fold_end); both 0 = all folds */
  int32_t fold_end;
  int32_t early_stop;      /* new: stop at the first checkpoint meeting the rule in DESIGN.md */
} pcvg_run_config;

/* Per-fold summary columns (FoldSummary engine.hpp:62-73 + FoldScore scoring.hpp:14-23). */
typedef struct {
  double* estimate;            /* [n_models*K] */
  double* log_f_hat;
  double* mc_contribution;
  double* naive_contribution;
  double* ess;
  double* rhat;                /* NaN when undefined */
  int64_t* batches;
  int32_t* fault;
  int32_t* failed;
  int32_t* dss_ridged;         /* FoldSummary::dss_ridged (engine.hpp:73); may be NULL */
} pcvg_fold_table;

/* pcv::PcvReport (engine.hpp:86-109). Arrays are caller-allocated; sizes in comments. */
typedef struct {
  pcvg_fold_table folds;       /* [n_models*K] each */
  int64_t* divergences;        /* [n_models*K*L] sampling-phase, task order */
  double* delta_k;             /* [K] */
  double* snapshots;           /* [n_checkpoints*7]: iteration, delta_hat, mcse,
                                  epistemic_se, prob_a_better, ess, rhat_max */
  double* benchmark;           /* [bench_draws] */
  /* outputs */
  double delta_hat, mcse, sigma2_delta, epistemic_se, prob_a_better, ess_overall, rhat_max;
  double score_total[2];
  int64_t numeric_faults[2];
  int32_t rhat_excluded[2];
  int64_t dropped_batch_draws;
  int32_t n_checkpoints;       /* written */
  int32_t benchmark_count;     /* written */
  int32_t verdict_pass;
  double verdict_quantile;
  double verdict_quantile_value;
  double verdict_observed;
  int64_t iters_run;           /* < iters when early stop fired */
  double warmup_ms;            /* device time of Step 2 */
  double sampling_ms;          /* device time of Step 3 */
  int64_t gpu_launches;        /* kernels launched by this call */
} pcvg_report;

typedef struct pcvg_ctx pcvg_ctx;

/* ---------------------------------------------------------------- version / errors */
int32_t pcvg_abi_version(void);
const char* pcvg_last_error(const pcvg_ctx* ctx); /* ctx may be NULL: thread-local last error */
const char* pcvg_status_name(int32_t status);

/* ---------------------------------------------------------------- host: RNG + folds
 * Bit-exact restatements of the reference's deterministic host pieces. */
uint64_t pcvg_stream_key(uint64_t kind, uint64_t a, uint64_t b, uint64_t c); /* rng.hpp:35-43 */
/* Draws from CounterRng(seed, stream), after skip_to(skip_block) when do_skip (rng.hpp:45-143). ops[i] in {'u','n','4' (next_u32),
 * 'b' (below(arg[i]))}; out[i] gets the draw as a double (u32/below as exact integers). */
pcvg_status pcvg_rng_sequence(uint64_t seed, uint64_t stream, int32_t do_skip, uint64_t skip_block,
                              const char* ops, const uint64_t* arg, int64_t n, double* out);
pcvg_status pcvg_make_loo(int64_t n_obs, int32_t* test_index, int32_t* K);          /* folds.cpp:43-52 */
pcvg_status pcvg_make_logo(const pcvg_dataset* d, int32_t* test_index, int32_t* K); /* folds.cpp:54-63 */
pcvg_status pcvg_make_kfold(int64_t n_obs, int32_t K, uint64_t seed, int32_t* test_index); /* folds.cpp:65-84 */
pcvg_status pcvg_make_time_blocks(const pcvg_dataset* d, int32_t K, int32_t* test_index); /* folds.cpp:86-108 */
/* hv-block (new): K contiguous test blocks in time order sized like time-blocks, training
 * excludes h ranks on each side. intervals: [K*4]. */
pcvg_status pcvg_make_hv_block(const pcvg_dataset* d, int32_t K, int64_t h, int64_t* intervals);
/* Racine (2000) per-point hv variant: fold t tests ranks [t-v, t+v], trains on |s-t| > v+h;
 * K = n_obs. */
pcvg_status pcvg_make_hv_racine(const pcvg_dataset* d, int64_t v, int64_t h, int64_t* intervals);

/* ---------------------------------------------------------------- host: simulators
 * Synthetic data generators (bit-exact restatements of the reference simulators, plus the
 * two new shapes). Output arrays are caller-allocated at the documented sizes. */
/* simulate_grouped_regression (grouped_regression.cpp:232-268): n = J*Nj. */
pcvg_status pcvg_simulate_grouped(int32_t J, int32_t Nj, int32_t P, double min_omitted_beta,
                                  uint64_t seed, double* y, double* x, int32_t* group_id);
/* simulate_radon_style (radon.cpp:216-240): n = houses, x = floor. */
pcvg_status pcvg_simulate_radon(int32_t houses, int32_t counties, uint64_t seed, double* y,
                                double* x, int32_t* group_id);
/* simulate_rat_growth (rat_growth.cpp:310-336): n = 5 * subjects, x = time. */
pcvg_status pcvg_simulate_rat(int32_t subjects, uint64_t seed, double* y, double* x, int32_t* group_id);
/* simulate_seasonal_ar (seasonal_ar.cpp:167-205): n = months - p, n_cov = p + q. */
pcvg_status pcvg_simulate_seasonal(int64_t months, int32_t p, int32_t q, double rho,
                                   double seasonal_amp, double sigma, uint64_t seed, double* y,
                                   double* x, int64_t* time_index);
/* cfg1/cfg5 linear regression: x ~ N(0,1), y = 0.5 + sum_p 0.3(p+1) x_p + N(0,1). */
pcvg_status pcvg_simulate_linreg(int64_t n, int32_t P, uint64_t seed, double* y, double* x,
                                 int32_t* group_id);
/* cfg2 logistic: x ~ N(0,1)/sqrt(P), beta* ~ N(0,1) (P+1 incl. intercept), y ~ Bern(sigmoid). */
pcvg_status pcvg_simulate_logistic(int64_t n, int32_t P, uint64_t seed, double* y, double* x);

/* ---------------------------------------------------------------- device context */
pcvg_status pcvg_create(int32_t device, pcvg_ctx** out);
pcvg_status pcvg_destroy(pcvg_ctx* ctx);

/* Registers one candidate model (at most two per run, engine.cpp:258-262): uploads the
 * dataset in the device layout, the fold masks, KernelParams and the full-data draw bank
 * (`_bank.f64` layout: bank_rows x dim row-major, report_io.cpp:159-167). model_id keys the
 * RNG streams (engine.cpp:299-309). Returns the model slot in *slot. */
pcvg_status pcvg_add_model(pcvg_ctx* ctx, const pcvg_dataset* data, const pcvg_folds* folds,
                           const pcvg_model_spec* spec, const pcvg_kernel* kernel,
                           const double* bank, int64_t bank_rows, int32_t model_id,
                           int32_t* slot);
pcvg_status pcvg_model_dim(const pcvg_ctx* ctx, int32_t slot, int32_t* dim);

/* Kernel selection. AUTO runs the Gaussian linear families (grouped, radon-style, seasonal AR, rat
 * growth) on fold sufficient statistics (SUFFSTAT below) when their data are finite. Otherwise, and always
 * under ROWS, the kernels stream the design matrix: the FP64 tensor-core GLM kernel for predictors
 * without group effects when enough chains (or a row-split cluster) fill the GPU, the
 * group-batched kernel for hierarchical models, else the generic lane-split kernel. GENERIC /
 * TENSOR force one of the row kernels (tests run every kernel). Logistic always uses the tensor
 * kernel. */
enum { PCVG_KERNEL_AUTO = 0, PCVG_KERNEL_GENERIC = 1, PCVG_KERNEL_TENSOR = 2, PCVG_KERNEL_TF32 = 3,
       PCVG_KERNEL_SUFFSTAT = 4, PCVG_KERNEL_ROWS = 5 };
/* PCVG_KERNEL_TF32: the FP32 variant of the logistic family: both contractions on
 * tcgen05 kind::tf32 with hi/lo-split operands (FP32-class accuracy, per-step values within 1e-5
 * of the FP64 path); chain state, energies and accumulators stay FP64. Other families ignore it. */
/* PCVG_KERNEL_SUFFSTAT: the Gaussian linear families (grouped, radon-style, seasonal AR) on fold
 * sufficient statistics: the masked sums of every gradient pass come from each fold's training
 * Gram matrix and group sums (built once on the host in double-double), O(d^2 + J d) per pass
 * instead of O(n d); same values to rounding. Needs finite data; other families
 * and non-finite datasets fall back to the ROWS choice. */
pcvg_status pcvg_set_kernel_policy(pcvg_ctx* ctx, int32_t policy);
/* Fault injection for tests (the reference's BrokenFoldModel, test_engine.cpp:57-90): every
 * transition of every chain of `fold` (0..K-1; -1 clears) in model `slot` is divergent, as when the
 * model's gradient is NaN on that fold. Exercises the failed-fold rule (engine.cpp:385-397). */
pcvg_status pcvg_debug_break_fold(pcvg_ctx* ctx, int32_t slot, int32_t fold);
pcvg_status pcvg_model_test_size(const pcvg_ctx* ctx, int32_t slot, int32_t fold, int64_t* n);

/* Parity probes (device). n evaluation points: fold[n], theta[n*dim]. */
/* Model::log_joint + grad_log_joint (model.hpp:34-36). */
pcvg_status pcvg_eval(pcvg_ctx* ctx, int32_t slot, int64_t n, const int32_t* fold,
                      const double* theta, double* log_joint, double* grad);
/* Model::log_pred (model.hpp:40). */
pcvg_status pcvg_eval_pred(pcvg_ctx* ctx, int32_t slot, int64_t n, const int32_t* fold,
                           const double* theta, double* log_pred);
/* hmc_step with injected momentum p0[n*dim] and uniform u[n] (hmc.cpp:53-99): returns the
 * new position, h0/h1, accepted/divergent flags. */
pcvg_status pcvg_hmc_probe(pcvg_ctx* ctx, int32_t slot, int64_t n, const int32_t* fold,
                           const double* theta, const double* momentum, const double* u,
                           double* theta_out, double* h0, double* h1, int32_t* accepted,
                           int32_t* divergent);
/* leapfrog (hmc.cpp:22-51) from (theta, momentum) with the model's kernel: the end point
 * (theta_out, momentum_out) of n_leapfrog steps; ok[c] = 0 where the trajectory went non-finite. */
pcvg_status pcvg_leapfrog(pcvg_ctx* ctx, int32_t slot, int64_t n, const int32_t* fold,
                          const double* theta, const double* momentum, double* theta_out,
                          double* momentum_out, int32_t* ok);
/* n_steps consecutive hmc_step calls of chain (fold, chain) on its own reference stream
 * CounterRng(seed, stream_key(ChainSampling, model_id, fold, chain)) from theta0: writes the
 * position after every step [n_steps*dim] and the divergence flags [n_steps]. */
pcvg_status pcvg_hmc_chain(pcvg_ctx* ctx, int32_t slot, int32_t fold, int32_t chain,
                           uint64_t seed, const double* theta0, int64_t n_steps,
                           double* trajectory, int32_t* divergent);

/* Online accumulators + fold reduction on explicit score streams: chain c feeds
 * s[c*n .. c*n+n) through ScoreAccum::observe (accum.cpp:164-182) with centre `center`, then the
 * fold is reduced by logs_fold_score + rhat_from_blocks (scoring.cpp:10-62, diagnostics.cpp:35-44).
 * out[8] = estimate, log_f_hat, mc_contribution, naive_contribution, ess, rhat, batches, fault. */
pcvg_status pcvg_score_streams(pcvg_ctx* ctx, int32_t L, int64_t n, const double* s, double center,
                               int32_t b, int32_t D, double* out);

/* ---------------------------------------------------------------- run (Steps 2-4) */
int32_t pcvg_checkpoint_count(const pcvg_run_config* cfg);
/* Full run_pcv on one device for the registered models. */
pcvg_status pcvg_run(pcvg_ctx* ctx, const pcvg_run_config* cfg, pcvg_report* report);

/* run_pcv's Steps 3-4 (checkpoints, per-fold statistics, shuffle benchmark, early-stop rule, report)
 * on given log_pred streams instead of sampled ones: chain c of fold k observes
 * s[(k*L + c)*iters + i] at iteration i through ScoreAccum::observe with centre centers[k]
 * (accum.cpp:164-182). One model, K folds, LogS, on a context with no models registered. The
 * harness of the reference's shuffle-benchmark acceptance criteria (acceptance.cpp:259-325, C6/C7)
 * through the same device accumulators, kernels and stopping rule as pcvg_run. */
pcvg_status pcvg_run_streams(pcvg_ctx* ctx, int32_t K, const double* s, const double* centers,
                             const pcvg_run_config* cfg, pcvg_report* report);

/* Stepwise API for fold-sharded multi-GPU runs (one process per GPU). */
/* Step 2 for the shard: warm start, warm-up, centering constants. */
pcvg_status pcvg_begin(pcvg_ctx* ctx, const pcvg_run_config* cfg);
/* Step 3 segment: n_iters more sampling iterations for every chain of the shard. */
pcvg_status pcvg_advance(pcvg_ctx* ctx, int64_t n_iters);
/* Per-fold LogS reductions of the shard at the current iteration (scoring.cpp:10-62,
 * diagnostics.cpp:35-44). Writes [n_models * shard_K] rows, model-major, into `out`
 * (estimate/log_f_hat/mc/naive/ess/rhat/batches/fault; failed = final failed-fold flag). */
pcvg_status pcvg_fold_stats(pcvg_ctx* ctx, pcvg_fold_table* out, int64_t* divergences,
                            int64_t* dropped_batch_draws, int64_t* iters_done);
/* Per-fold centred block sums for the shuffle benchmark: y_x/y_x2 [n_models*shard_K*L*D]. */
pcvg_status pcvg_block_sums(pcvg_ctx* ctx, double* y_x, double* y_x2);
/* Device event time of the last pcvg_advance call (ms) and kernel count so far. */
pcvg_status pcvg_timing(const pcvg_ctx* ctx, double* last_advance_ms, int64_t* launches);
/* Device time of the current run's Step 2 (pcvg_begin) and of its Step-3 advances so far (ms). */
pcvg_status pcvg_phase_times(const pcvg_ctx* ctx, double* warmup_ms, double* sampling_ms);

/* Host merge (Step 4, engine.cpp:117-253 + 385-480): from the full (all-shard, fold-order)
 * per-fold tables produce the global statistics. `final_checkpoint` applies the failed-fold
 * exclusions (engine.cpp:415-418). y_x/y_x2 may be NULL to skip the benchmark. */
pcvg_status pcvg_merge(int32_t n_models, int32_t K, const pcvg_run_config* cfg,
                       int64_t iter_count, int32_t final_checkpoint,
                       const pcvg_fold_table* folds, const double* y_x, const double* y_x2,
                       pcvg_report* report);

/* ---------------------------------------------------------------- Step 1: full-data fit
 * adapt_full_data (adapt.hpp:64-69, adapt.cpp:96-221) on the device: L_fd chains from the model's
 * prior (Model::initial_draw on CounterRng(seed, stream_key(FullData, model_id, c)), host), the
 * StepInit doubling search for the first step size, dual-averaging step-size adaptation
 * (adapt.hpp:15-44) with windowed diagonal mass estimation on the full-data sentinel fold, then
 * `draws` frozen-kernel transitions that fill the warm-start bank. Every transition of every chain
 * runs in the fused HMC kernels; the window / dual-averaging arithmetic (a few doubles per
 * iteration) stays on the host, as in the reference coordinator. */
typedef struct {
  int32_t chains;          /* L_fd */
  int64_t warmup;
  int64_t draws;
  int32_t n_leapfrog;
  double target_accept;
  double init_step_size;   /* 0 = StepInit search */
} pcvg_adapt_config;       /* AdaptConfig, adapt.hpp:47-54 */

typedef struct {
  double step_size;
  double* inv_mass_diag;   /* [dim] */
  double* draws;           /* [chains*draws*dim]: row iter*chains + chain (adapt.cpp:204-209) */
  double* rhat;            /* [dim] param_rhat (adapt.cpp:45-66), may be NULL */
  double* ess;             /* [dim] param_ess (adapt.cpp:69-92), may be NULL */
  double* step_trace;      /* [warmup] step size used at each warm-up iteration, may be NULL */
  int64_t divergences;     /* sampling phase */
  double mean_accept;
  double device_ms;        /* device time of all transitions */
} pcvg_fit;                /* FullDataFit, adapt.hpp:56-62 */

/* Model::initial_draw (model.hpp:44) on CounterRng(seed, stream): host, bit-exact. */
/* Host-only probe of the sufficient-statistics kernel's fold statistics: for rows
 * with y[n], x[nc][n] (column-major) and fold keys key[n], fold k (0..K-1) holding out rows with
 * lo[k] <= key < hi[k], writes the packed lower triangle of sum u u^T over each fold's training
 * rows, u = (y, x), to gram[(K+1) * (nc+1)(nc+2)/2] (index K = all rows). Returns
 * PCVG_INVALID_INPUT when the data are not finite (the kernel then keeps the row kernels). */
pcvg_status pcvg_fold_gram(int64_t n, int32_t nc, const double* y, const double* x, const int32_t* key,
                           int32_t K, const int32_t* lo, const int32_t* hi, double* gram);
pcvg_status pcvg_initial_draw(const pcvg_dataset* data, const pcvg_folds* folds,
                              const pcvg_model_spec* spec, uint64_t seed, uint64_t stream,
                              double* theta);
pcvg_status pcvg_adapt_full_data(pcvg_ctx* ctx, const pcvg_dataset* data, const pcvg_folds* folds,
                                 const pcvg_model_spec* spec, const pcvg_adapt_config* cfg,
                                 uint64_t seed, int32_t model_id, pcvg_fit* out);

/* Shuffle benchmark (diagnostics.cpp:76-101, engine.cpp:464-480) of this context's shard on
 * device. Replicate r consumes CounterRng(seed, stream_key(Benchmark, r, 0, 0)) sequentially over
 * (model, non-failed fold, chain, block), one below(L) each; this shard's non-failed folds are
 * global items m * nonfailed_total + nonfailed_before + j. failed: [shard folds] or NULL (none).
 * rep_max[bench_draws]: max R-hat over the shard's items (0 = none; all-reduce MAX across shards);
 * needs_host[bench_draws]: 1 where a below() rejection (probability < L / 2^64 per draw) makes the
 * positional stream differ from the sequential one - run the sequential host path for it. */
pcvg_status pcvg_benchmark(pcvg_ctx* ctx, const int32_t* failed, int64_t nonfailed_before,
                           int64_t nonfailed_total, int32_t blocks_used, double* rep_max,
                           int32_t* needs_host);
/* The same positional benchmark on host sub-block sums y_x/y_x2 [n_models][nfold][L][D_stride]
 * (multi-process CPU tests of the sharding arithmetic): the first blocks_used sub-blocks regrouped
 * into block_groups benchmark blocks (pcvg_benchmark uses min(RunConfig blocks, blocks_used)). */
pcvg_status pcvg_benchmark_host(int32_t n_models, int32_t nfold, int32_t L, int32_t D_stride,
                                int32_t blocks_used, int32_t block_groups, int64_t iter_count, uint64_t seed,
                                int32_t bench_draws, const double* y_x, const double* y_x2,
                                const int32_t* failed, int64_t nonfailed_before,
                                int64_t nonfailed_total, double* rep_max, int32_t* needs_host);
/* pcvg_merge with precomputed benchmark replicate maxima (all shards reduced by MAX). */
pcvg_status pcvg_merge_bench(int32_t n_models, int32_t K, const pcvg_run_config* cfg,
                             int64_t iter_count, int32_t final_checkpoint,
                             const pcvg_fold_table* folds, const double* bench_max,
                             pcvg_report* report);

/* ---------------------------------------------------------------- multi-GPU (one process)
 * run_pcv with the folds sharded across devices: one context per device, device i
 * owning folds [i K / n, (i + 1) K / n) with all L chains of each fold; each device advances on its own
 * host thread, the per-fold tables are merged in fold order at every check interval and the shuffle
 * benchmark runs on each device's block sums at its global stream offset (replicate maxima combined
 * by MAX), so the statistics do not depend on the device count. Implemented above this ABI with the
 * stepwise calls (csrc/multi_device.cpp). A device id may repeat (several shards on one GPU). */
typedef struct pcvg_multi pcvg_multi;
pcvg_status pcvg_multi_create(int32_t n_devices, const int32_t* devices, pcvg_multi** out);
pcvg_status pcvg_multi_destroy(pcvg_multi* mc);
const char* pcvg_multi_last_error(const pcvg_multi* mc);
pcvg_status pcvg_multi_add_model(pcvg_multi* mc, const pcvg_dataset* data, const pcvg_folds* folds,
                                 const pcvg_model_spec* spec, const pcvg_kernel* kernel, const double* bank,
                                 int64_t bank_rows, int32_t model_id, int32_t* slot);
pcvg_status pcvg_multi_set_kernel_policy(pcvg_multi* mc, int32_t policy);
pcvg_status pcvg_multi_run(pcvg_multi* mc, const pcvg_run_config* cfg, pcvg_report* report);

#ifdef __cplusplus
}
#endif
#endif /* PCVG_H */
