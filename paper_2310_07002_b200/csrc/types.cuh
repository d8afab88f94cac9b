// Device-side descriptors of one uploaded model and of its chains.
#pragma once
#include <cstdint>

#include "device_common.cuh"

namespace pcvg {

// Device family codes: pcvg_family, with the rat-growth model split by slope structure.
enum Family : int { kGrouped = 0, kRadon = 1, kSeasonal = 2, kLogistic = 3, kRatB = 4, kRatA = 5 };

// Kernel modes.
enum Mode : int {
  kModeEval = 0,    // gradient + log joint at the stored position (init, pcvg_eval)
  kModeWarmup = 1,  // Step 2: hmc steps, Sigma log_pred into warm_sum (hmc.cpp:121-149)
  kModeSample = 2,  // Step 3: hmc steps, ScoreAccum::observe (engine.cpp:342-381)
  kModeProbe = 3,   // one hmc step with injected momentum / uniform (parity probe)
  kModeChain = 4,   // hmc steps recording every (transition, chain): position, flags, h0, h1
                    // (parity probe, full-data adaptation)
  kModePred = 5     // log_pred at the stored position (parity probe)
};

constexpr int kMaxCov = 16;

struct ModelDev {
  int family;
  int n;     // observations (device row order: group-major for hierarchical families)
  int nc;    // covariate columns read by the kernel
  int J;     // groups (the first J dims are one parameter per group; kRatA: 2J dims)
  int goff;  // index of the first global parameter (J, or 2J for kRatA)
  int ng;    // global parameters (dims J..dim-1)
  int dim;
  int K;     // folds; index K is the full-data sentinel
  const double* y;    // [n]
  const double* x;    // [nc][n] column-major (coalesced per covariate)
  const double* xr;   // [n][nc_pad] row-major copy (logistic tiles), may be null
  int nc_pad;
  const int* key;     // [n] partition fold id, or time rank (hv-block)
  const int* grp_ptr; // [J+1]
  const int* fold_lo; // [K+1] row i is held out of training iff lo <= key[i] < hi
  const int* fold_hi;
  const int* n_train; // [K+1]
  const int* fold_seg;  // [K+2] test segments of fold k: [fold_seg[k], fold_seg[k+1])
  const int* seg_group;
  const int* seg_unseen;
  const int* seg_row;   // [nseg+1]
  const int* seg_rows;  // device row ids of the test rows
  const double* inv_mass;  // [dim]
  double step;
  int n_lf;
  // family options and host-computed prior constants (glibc lgamma/log, priors.hpp:13-26)
  double cmask[kMaxCov];  // grouped covariate mask as 0/1
  int include_floor;
  int p, q, rho_sym;
  double c_lhn10, c_lhn1;  // 0.5 log(2/(pi v)) for v = 10, 1
  double c_lgamma6_9;      // 6 log 9 - lgamma(6)
  double c_lgamma10_10;    // 10 log 10 - lgamma(10)
  double c_lbeta55;        // lgamma(10) - 2 lgamma(5)
  double c_log4;           // log(4)
  double c_lg25_2, c_lg5_10, c_lg1_2;  // a log r - lgamma(a): Gamma(25,2), Gamma(5,10), Gamma(1,2)
  double c_log20, c_log2;              // log 20, log 2 (rat-growth normal hyper-priors)
  // group-batched layout (hierarchical families, gauss_kernel NB > 0): nb batches of 32 group
  // slots; bgroup[b*32 + i] = group of lane i in batch b (-1 = none); rows of batch b are
  // [boff[b], boff[b+1]) in lane-interleaved arrays (row j of lane i at j*32 + i), padded with
  // key -1 rows; bstride = boff[nb] (rows per lane).
  int nb;
  int bstride;
  const int* bgroup;
  const int* boff;
  const double* yb;
  const double* xb;  // [nc][bstride*32]
  const int* keyb;
  // row tiles of a pass (at most rt rows each, batch order): tile_first[b] .. tile_first[b+1]
  int ntile;
  int rt;
  const int* tile_first;  // [nb+1]
  const int* tile_r0;     // [ntile] first row (batch layout)
  const int* tile_rows;   // [ntile]
  int bkey_uniform;       // every group's rows share one fold key (LOGO): per-slot key below
  const int* bkey;        // [nb*32] the group's key (-1 = no group)
  const int* bgrows;      // [nb*32] the group's row count
  const int* buniform;    // [nb] 1 if every group of the batch has the batch's row count
  int ring;               // 1: row tiles staged through a shared-memory TMA ring; 0: read via L1
  const unsigned char* x32;  // logistic FP32 variant: TF32-split tile images (glm32_kernel.cu)
  // fold sufficient statistics of the Gaussian families (suffstats.cpp, gauss_kernel NB < 0):
  // u = (y, x_0..x_{nc-1}); sA[k] = packed lower sum of u u^T over fold k's training rows;
  // sgn / sgs full-data group counts / sums of u; fold k overrides groups sov_g[sov_ptr[k] ..
  // sov_ptr[k+1]) with (sov_n, sov_s); its excluded rows are sex_rows[sex_lo[k] .. sex_hi[k]).
  int suff;  // 1 if the statistics exist
  int sd, sdp;
  const double* sA;
  const double* sgn;
  const double* sgs;
  const int* sov_ptr;
  const int* sov_g;
  const double* sov_n;
  const double* sov_s;
  const int* sex_lo;
  const int* sex_hi;
  const int* sex_rows;
  const int* sex_grp;
  double* g32_scratch;  // logistic FP32 variant: per-CTA FP64 G partials (the model's own buffer)
  double su[kMaxCov + 1];  // centre ubar of u = (y, x): sA / sgs / sov_s are statistics of u - ubar
  const double* sgA;    // rat M_A: [J][3] full-data per-group (y, t) Gram (yy, ty, tt)
  const double* sov_A;  // rat M_A: [nov][3] the fold's override Grams
  // fault injection (tests only, pcvg_debug_break_fold): every transition of a chain of this fold is
  // divergent, as with the reference's BrokenFoldModel whose gradient is NaN on one fold
  // (test_engine.cpp:57-90); -1 = none
  int broken_fold;
  int any_unseen;
  // few-chain GLM launches split over several clusters per chain tile (glm_kernel.cu): cluster
  // partials [tile][parity][cluster][KP*64 + 64] and per-tile arrival counters (the model's buffers)
  double* glm_part;
  unsigned int* glm_cnt;  // some fold holds out every row of a group (compound predictive needed)
};

constexpr int kMaxBatches = 16;

// Kernel launches issued by the sampler launchers on this host thread (a wave-tail split issues
// two); the driver adds the difference around each launch to its launch count.
inline int& sampler_launch_count() {
  static thread_local int n = 0;
  return n;
}

// HS / DSS score state (ScoreKind::HS / DSS, engine.cpp:322-373; accum.cpp:10-99). Per local fold
// kf with test size m = msize[kf], the L chains of the fold are interleaved entry-major: entry e of
// chain cl sits at base[kf] + e * L + cl (one 8*L-byte segment per entry).
//   HS : acc  e in [0,2m) WelfordDiag a_x of xi = (d2 + d1^2, d1), [2m,4m) a_x2
//        warm [0,m) hs1_sum, [m,2m) hs2_sum (WarmupStats, hmc.cpp:133-140); centre 2m per fold
//   DSS: acc  [0,m) WelfordAccumulator a_x, then the packed lower triangle a_xx (row i: i+1 entries)
//        warm [0,m) pred_sum; dev [0,m) staging of x - c for the triangle update; centre m per fold
// The observation count is the ScoreAccum count (both advance once per sampling iteration).
struct ExtraDev {
  int kind;              // pcvg_score: 0 = LogS (no extra state), 1 = HS, 2 = DSS
  const int* msize;      // [nfold] test size
  const int64_t* base;   // [nfold] accumulator base
  const int64_t* wbase;  // [nfold] warm-up sum / staging base
  const int64_t* cbase;  // [nfold] centre base
  double* acc;
  double* warm;
  double* dev;
  double* center;
};

struct ChainsDev {
  int nch;        // chains on this device (task order restricted to the shard)
  int L;          // chains per fold
  int fold0;      // first global fold of the shard
  const int* fold_override;  // probes: explicit fold per chain, or null
  uint64_t seed;
  uint64_t stream_model;  // model id used in stream keys (0 under shared_streams)
  double* pos;    // [2][dim][nch] position (double buffered, `cur` selects)
  double* grad;   // [2][dim][nch] cached gradient at pos
  double* wp;     // [dim][nch] working momentum (group dims) / probe scratch
  double* lp0;    // [nch] cached log joint at pos
  int8_t* cur;    // [nch]
  uint64_t* rng_stream;  // [nch] stream_key(ChainSampling, model, fold, chain)
  uint64_t* rng_pos;
  double* rng_cached;
  int8_t* rng_has;
  int64_t* divergences;  // cumulative (warm-up + sampling), hmc.hpp:20-24
  double* warm_sum;      // WarmupStats::logpred_sum
  AccumDev acc;
  ExtraDev X;
  double* probe_p_out;  // leapfrog probe: final momentum [nch][dim] of group dims (batched kernel)
};

struct RunArgs {
  int mode;
  int64_t n_iters;
  int64_t iter0;      // sampling iteration index of the first step (block_for)
  int64_t planned_n;  // N (accum.hpp:96-111)
  int D;
  int b;
  const double* probe_momentum;  // [nch][dim]
  const double* probe_u;         // [nch]
  double* out_a;  // probe: h0 / eval: log joint / pred: log_pred   [nch]
  double* out_b;  // probe: h1                                      [nch]
  int32_t* out_flags;  // probe: accepted | divergent << 1           [nch]
  double* traj;        // chain mode: [n_iters][nch][dim] or null
  int32_t* traj_div;   // chain mode: [n_iters][nch] accepted | divergent << 1, or null
};

}  // namespace pcvg
