/*
 * TEST INFRASTRUCTURE ONLY - the CPU oracle for the PCV hot path.
 *
 * A plain-C restatement of the reference algorithm (/root/reference/proj) for the path
 * BASELINE.json's north_star names: Philox streams, fold schemes, the masked model
 * evaluations of every on-path family, leapfrog/hmc_step, the online accumulators, Steps 2-3
 * of run_pcv and the Step-4 reductions. Every function cites the reference file:line it
 * follows. It is pinned against (a) the reference's own golden vectors (Philox KATs, R-hat and
 * selection-probability closed forms, ...) and (b) the reference itself compiled in place
 * (oracle/_ref/libpcvref.so) - see tests/test_oracle_*.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library. The product (paper_2310_07002_b200/, libpcvg.so) never does.
 */
#ifndef PCV_ORACLE_H
#define PCV_ORACLE_H

#include <stdint.h>

#include "../include/pcvg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* CounterRng, rng.hpp:45-143. */
typedef struct {
  uint32_t key[2], ctr[4], buf[4];
  int have;
  double cached;
  int has_cached;
} pcvo_rng;

void pcvo_rng_init(pcvo_rng* r, uint64_t seed, uint64_t stream);
uint32_t pcvo_next_u32(pcvo_rng* r);
uint64_t pcvo_next_u64(pcvo_rng* r);
double pcvo_uniform(pcvo_rng* r);
double pcvo_normal(pcvo_rng* r);
uint64_t pcvo_below(pcvo_rng* r, uint64_t n);
void pcvo_skip_to(pcvo_rng* r, uint64_t block);
uint64_t pcvo_stream_key(uint64_t kind, uint64_t a, uint64_t b, uint64_t c);
int pcvo_rng_sequence(uint64_t seed, uint64_t stream, int32_t do_skip, uint64_t skip_block,
                      const char* ops, const uint64_t* arg, int64_t n, double* out);

/* Fold schemes, folds.cpp:43-108, plus hv-block (new). Return 0 on success. */
int pcvo_make_kfold(int64_t n, int32_t K, uint64_t seed, int32_t* out);
int pcvo_make_time_blocks(const pcvg_dataset* d, int32_t K, int32_t* out);
int pcvo_make_hv_block(const pcvg_dataset* d, int32_t K, int64_t h, int64_t* intervals);
int pcvo_make_hv_racine(const pcvg_dataset* d, int64_t v, int64_t h, int64_t* intervals);

/* Models (opaque). */
typedef struct pcvo_model pcvo_model;
void pcvo_model_break_fold(pcvo_model* m, int32_t fold);
pcvo_model* pcvo_model_create(const pcvg_dataset* d, const pcvg_folds* f,
                              const pcvg_model_spec* s);
void pcvo_model_destroy(pcvo_model* m);
int32_t pcvo_model_dim(const pcvo_model* m);
int64_t pcvo_test_size(const pcvo_model* m, int32_t fold);
double pcvo_log_joint(const pcvo_model* m, const double* theta, int32_t fold);
void pcvo_grad(const pcvo_model* m, const double* theta, int32_t fold, double* grad);
double pcvo_log_pred(const pcvo_model* m, const double* theta, int32_t fold);

/* Model::pred_derivs / pred_sample over the fold's test rows (model.hpp:54-66); the logistic
 * family supports neither (pcvo_supports_pred = 0). */
int pcvo_supports_pred(const pcvo_model* m);
void pcvo_pred_derivs(const pcvo_model* m, const double* theta, int32_t fold, double* d1, double* d2);
void pcvo_pred_sample(const pcvo_model* m, const double* theta, int32_t fold, pcvo_rng* rng, double* out);
/* `times` consecutive pred_sample calls on one CounterRng(seed, stream): out[times * test_size]. */
int pcvo_pred_sample_stream(const pcvo_model* m, const double* theta, int32_t fold, uint64_t seed,
                            uint64_t stream, int32_t times, double* out);

/* hmc.cpp:22-99. */
int32_t pcvo_leapfrog(const pcvo_model* m, int32_t fold, double step, int32_t n_lf,
                      const double* inv_mass, double* q, double* p);
/* hmc_step with injected momentum and uniform (the RNG draws replaced by inputs). */
void pcvo_hmc_probe(const pcvo_model* m, int32_t fold, double step, int32_t n_lf,
                    const double* inv_mass, const double* theta, const double* momentum,
                    double u, double* theta_out, double* h0, double* h1, int32_t* accepted,
                    int32_t* divergent);
int pcvo_hmc_chain(const pcvo_model* m, int32_t fold, double step, int32_t n_lf,
                   const double* inv_mass, uint64_t seed, uint64_t stream,
                   const double* theta0, int64_t n_steps, double* traj, int32_t* divergent);

/* Per-task end state of Steps 2-3 (engine.cpp:295-381), task order (m*K+k)*L+c.
 * accum row per task: [u_x, u_x2, z_x, v_x, v_x2, committed, pending, count, faults, c,
 *                      y_x[D], y_x2[D]]  (10 + 2D doubles). */
typedef struct {
  double* position;        /* [tasks*dim_max] (dim of the task's model, padded) */
  double* warm_logpred;    /* [tasks] */
  int64_t* divergences;    /* [tasks] sampling-phase */
  double* accum;           /* [tasks*(10+2D)] */
} pcvo_task_out;

/* run_pcv (engine.cpp:257-483): n_models in {1,2}. threads <= 0 = all cores.
 * tasks may be NULL. Returns a pcvg_status. */
int pcvo_run_pcv(int32_t n_models, pcvo_model** models, const int32_t* model_ids,
                 const pcvg_kernel* kernels, const double* const* banks,
                 const int64_t* bank_rows, const pcvg_run_config* cfg, int32_t threads,
                 pcvg_report* rep, pcvo_task_out* tasks, int32_t dim_max);

/* Step-4 pieces for unit pinning (scoring.cpp, diagnostics.cpp). */
int pcvo_rhat_from_sums(const double* sx, const double* sxx, int32_t l, int64_t n,
                        double* w, double* b, double* rhat);
double pcvo_selection_probability(double delta_hat, const double* deltas, int64_t k,
                                  double* sigma2);
double pcvo_benchmark_quantile(const double* values, int64_t n, double q);

/* Steps 2-3 task loop on a fold sample (bench CPU baseline, kind "port"). */
int pcvo_time_tasks(const pcvo_model* m, int32_t n_folds, const int32_t* folds, int32_t L,
                    int64_t warmup, int64_t iters, uint64_t seed, int32_t model_id,
                    const pcvg_kernel* k, const double* bank, int64_t bank_rows, int32_t threads,
                    double* sampling_s, double* warmup_s, double* checksum);

/* Online accumulators + fold reduction on explicit score streams (accum/scoring/diagnostics). */
int pcvo_score_streams(int32_t L, int64_t n, const double* s, double center, int32_t b, int32_t D,
                       double* out);

const char* pcvo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
