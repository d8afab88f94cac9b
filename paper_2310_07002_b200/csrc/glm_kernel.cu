// Fused HMC kernel on FP64 tensor cores for every family whose per-observation predictor is a
// GEMM across chains (sm_100a):
//   logistic  (new family, BASELINE configs[1])          eta = X . theta,       r = y - sigmoid(eta)
//   grouped regression with one group (cfg1, cfg5)       eta = alpha + X . beta, r = y - eta
//       (grouped_regression.cpp:56-122 with J = 1)
//   seasonal AR (cfg4; seasonal_ar.cpp:37-105)           eta = b0 + sum rho(u) lag + sum b d
// For the 64 chains of a CTA and every gradient pass over N observations:
//   eta = X_tile . W  ->  R = mask(y - mean(eta))  ->  G += X_tile^T . R
// with X = [1, covariates] ([N][KP] row-major, KP in {8, 16, 52}), W the per-chain GEMM weights
// (a family transform of the parameters), both contractions on DMMA (mma.sync.m8n8k4.f64). X row
// tiles stream through a 3-stage TMA bulk-copy ring guarded by full/empty mbarriers; 16 warps =
// 4 row quarters x 4 chain groups, each reading back only its own R block so warps drift and
// overlap phases. Parameters live in shared memory, momenta in the registers of 8 owner threads per
// chain, which also apply the family chain rule (gradient in parameter space from G, the residual
// sum of squares and the priors). One chain thread per chain runs the reference RNG stream,
// energies, Metropolis test, log_pred and accumulators. Semantics follow hmc.cpp:22-99 and
// engine.cpp:342-381.
// Few-chain configurations (K-fold cfg2: 80 chains; Step 1: one tile) split the rows over
// thread-block clusters of CS CTAs that replicate one 64-chain tile, and over NC such clusters
// (cooperative launch): each CTA streams its share of the row tiles; the partial X^T R / residual
// sums are reduced by a push over DSMEM (bulk copies to row owners, rank-order sums, bulk copies
// back; reduce_pass) and, across clusters, through global memory (reduce_clusters), so every CTA
// of the tile holds bit-identical state; rank 0 writes it back. The wave tail of many-chain launches
// runs the same way (clusters only). log_pred's test rows are split over the first cluster's ranks.
#include <algorithm>
#include <mutex>
#include <cooperative_groups.h>
#include <cuda/atomic>
#include <cstdio>
#include <cstdlib>
#include <math_constants.h>

#include "device_cache.hpp"
#include "device_common.cuh"
#include "score_extra.cuh"
#include "tc_common.cuh"
#include "types.cuh"

namespace pcvg {

int glm_cluster_size(int n, int kp, int nch);
int glm_sm_count();
int glm_clusters_per_tile(int n, int kp, int nch, int cs, bool have_scratch);

namespace {

using namespace tc;

constexpr int kC = 64;          // chains per CTA
constexpr int kLdS = 68;        // leading dim of [k][chain] / [row][chain] shared arrays
constexpr int kMaxOwners = 8;   // owner threads per chain at 512 threads
constexpr int kStages = 3;      // TMA ring depth
constexpr int kMaxClusters = 16;  // clusters per chain tile in multi-cluster launches

// Warp layout: 4 chain groups (16 chains each) x RQ row groups. WREG (tested for KP = 52 with 8 warps
// of 250 registers holding each warp's GEMM-weight fragments for the whole pass) ran 3% slower than
// 16 warps of 128 registers: with two warps per scheduler the sigmoid phases no longer hide behind
// other warps' DMMA (profiles/r02_glm_layout.log; ncu's "shared pipe" is the FP64 datapath that
// DMMA and DFMA share, not shared memory). So every design runs 16 warps.
template <int KP, int THREADS_ = 512>
struct Geom {
  static constexpr int THREADS = THREADS_;
  static constexpr int WARPS = THREADS / 32;
  static constexpr int RQ = WARPS / 4;                    // row groups
  static constexpr int OWNERS = THREADS / kC;             // owner threads per chain
  static constexpr bool WREG = THREADS_ < 512;            // weight fragments in registers
  static constexpr int KS = KP / 4;                       // k-steps of X . W
  static constexpr int PT = (KP + 7) / 8;                 // 8-row tiles of X^T . R
  static constexpr int TM = KP <= 8 ? 256 : (KP <= 16 ? 128 : 64);  // rows per TMA tile
  static constexpr int ROWS_W = TM / RQ;                  // rows per warp per tile
  static constexpr int CHUNKS = ROWS_W / 16;              // 16-row chunks per warp per tile
  static constexpr int XPAD = PT * 8 - KP + 4;            // X^T p-tile overread
  static constexpr int DIMP = KP + 4;                     // max parameters (incl. specials)
  static constexpr int OWN = (DIMP + OWNERS - 1) / OWNERS;
  static constexpr int TILE_BYTES = TM * KP * 8 + TM * 8 + TM * 4;
  // reduced rows: G [col][chain] rows 0..KP-1 and the residual statistic as row KP, in sm.rs
  static constexpr int RROWS = KP + 1;
  // receive scratch rows of a cluster reduction: (cs - 1) partials of ceil(RROWS / cs) rows, any cs <= 16
  static constexpr int scr_rows() {
    int m = 0;
    for (int c = 2; c <= 16; ++c) {
      const int v = (c - 1) * ((RROWS + c - 1) / c);
      m = v > m ? v : m;
    }
    return m;
  }
  static constexpr int SCR = scr_rows();
  static_assert(RROWS <= 64, "the reduced rows live in sm.rs (64 rows)");
};

// Residual statistic of chain c summed over the row groups in a fixed tree order.
template <int RQ>
__device__ __forceinline__ double rq_sum(const double (*llp)[kC], int c) {
  if constexpr (RQ == 4) return (llp[0][c] + llp[1][c]) + (llp[2][c] + llp[3][c]);
  else if constexpr (RQ == 2) return llp[0][c] + llp[1][c];
  else return llp[0][c];
}

template <int KP>
struct Smem {
  using G = Geom<KP>;
  double xs[kStages][G::TM * KP + G::XPAD];
  double ys[kStages][G::TM];
  int ks[kStages][G::TM];
  double rs[(KP > 64 ? KP : 64) * kLdS];  // per-warp R blocks; reused as G and momentum staging
  double qs[G::DIMP * kLdS];              // parameters, [k][chain]
  double im[G::DIMP];                     // inverse mass (shared memory: the device-scope acquire of the
                                          // multi-cluster reduction invalidates L1 every pass)
  double ws[KP * kLdS];                   // GEMM weights, [col][chain]
  double llp[4][kC];                      // per row group: log-lik (logistic) / sum r^2 (gaussian)
  double gt[G::SCR * kLdS];               // cluster reduction: partial rows received from the other ranks
  double red[kMaxOwners][kC];             // owner partial sums (kinetic)
  double lpp[kC];                         // this rank's log_pred partial per chain (cluster ranks split rows)
  unsigned long long rng_pos[kC];         // momentum draws: each chain's stream position,
  double rng_cached[kC], rng_tail[kC];    // cached normal in / out,
  int rng_has[kC];                        // and cached flag at the transition start
  double pri[kMaxOwners][kC];             // owner partial sums (log joint)
  double exp_tab[16];                     // 2^(-j/16)
  double l1p_rc[64], l1p_lc[64];          // log1p_01: 1 / c_j and log(c_j), c_j = 1 + (j + 1/2) / 64
  int exp_hi32[32], exp_lo32[32];          // 2^(-j/32) as high / low words (gradient-only sigmoid)
  int lo[kC], hi[kC], ntr[kC];
  int bad[kC];
  int cur[kC];
  int fold[kC];                           // the chain's fold (K for padding chains)
  unsigned long long full[kStages];
  unsigned long long rbar[2];  // cluster reduction: partials received (0), reduced rows gathered (1)
  unsigned int rel[kStages];  // warps done with each ring slot (monotonic; last arrival refills)
};
static_assert(sizeof(Smem<52>) <= 227 * 1024, "one CTA per SM: at most 227 KB of shared memory");

// ------------------------------------------------------------------ family hooks
__device__ __forceinline__ double logistic_fn(double u) { return 1.0 / (1.0 + exp(-u)); }

// Design column of parameter k, or -1 for parameters outside the predictor.
template <int FAM>
__device__ __forceinline__ int col_of(const ModelDev& M, int k) {
  if constexpr (FAM == kLogistic) return k < M.dim ? k : -1;
  else if constexpr (FAM == kGrouped) return k <= M.nc ? k : -1;  // [alpha_0, beta_0..beta_{P-1}]
  else return k < M.p ? k + 1 : (k == M.p ? 0 : (k <= M.p + M.q ? k : -1));
}

// GEMM weight of parameter k (the coefficient multiplying its design column).
template <int FAM>
__device__ __forceinline__ double w_of(const ModelDev& M, int k, double qk) {
  if constexpr (FAM == kGrouped) return k == 0 ? qk : M.cmask[k - 1] * qk;
  else if constexpr (FAM == kSeasonal) {
    if (k < M.p) {
      const double w = logistic_fn(qk);
      return M.rho_sym ? 2.0 * w - 1.0 : 0.5 * (1.0 + w);
    }
    return qk;
  } else return qk;
}

template <int KP>
__device__ __forceinline__ double quarter_sum(const Smem<KP>& sm, int c) {
  return sm.rs[KP * kLdS + c];  // reduced over row quarters and cluster ranks (reduce_pass)
}

// d log p / d q_k from the reduced G column, the parameters and the residual sum of squares.
// grouped_regression.cpp:100-121 (J = 1), seasonal_ar.cpp:79-105, logistic plugin.
template <int FAM, int KP>
__device__ __forceinline__ double grad_of(const ModelDev& M, const Smem<KP>& sm, int k, int c,
                                          double gk, double qk) {
  if constexpr (FAM == kLogistic) {
    return gk - qk;
  } else if constexpr (FAM == kGrouped) {
    const int P = M.nc;
    const double sig_y = exp(sm.qs[(P + 3) * kLdS + c]);
    const double v = sig_y * sig_y;
    const double sig_a = exp(sm.qs[(P + 2) * kLdS + c]);
    const double va = sig_a * sig_a;
    const double mu = sm.qs[(P + 1) * kLdS + c];
    const double dev = sm.qs[c] - mu;
    if (k == 0) return gk / v - dev / va;
    if (k <= P) return M.cmask[k - 1] * (gk / v) - qk;
    if (k == P + 1) return dev / va - mu;
    if (k == P + 2) return dev * dev / va - 1.0 - va / 10.0 + 1.0;
    return quarter_sum(sm, c) / v - sm.ntr[c] - v / 10.0 + 1.0;
  } else {
    const int p = M.p, q = M.q;
    const double sigma = exp(sm.qs[(p + q + 1) * kLdS + c]);
    const double v = sigma * sigma;
    if (k < p) {
      const double w = logistic_fn(qk);
      const double dw = w * (1.0 - w);
      const double drho = M.rho_sym ? 2.0 * dw : 0.5 * dw;
      return gk * drho / v + (4.0 * (1.0 - w) - 4.0 * w + 1.0 - 2.0 * w);
    }
    if (k <= p + q) return gk / v - qk;
    return quarter_sum(sm, c) / v - sm.ntr[c] - v + 1.0;
  }
}

// Log joint contribution owned by parameter k (priors; the Gaussian likelihood term rides on the
// observation-variance parameter). grouped_regression.cpp:65-85, seasonal_ar.cpp:59-77.
template <int FAM, int KP>
__device__ __forceinline__ double logp_of(const ModelDev& M, const Smem<KP>& sm, int k, int c,
                                          double qk) {
  if constexpr (FAM == kLogistic) {
    return -0.5 * (kLog2Pi + qk * qk);
  } else if constexpr (FAM == kGrouped) {
    const int P = M.nc;
    if (k == 0) {
      const double sig_a = exp(sm.qs[(P + 2) * kLdS + c]);
      const double va = sig_a * sig_a;
      const double dev = qk - sm.qs[(P + 1) * kLdS + c];
      return -0.5 * (kLog2Pi + log(va) + dev * dev / va);
    }
    if (k <= P + 1) return -0.5 * (kLog2Pi + qk * qk);
    const double s = exp(qk);
    double l = M.c_lhn10 - s * s / 20.0 + qk;
    if (k == P + 3) {
      const double v = s * s;
      l += -0.5 * (sm.ntr[c] * (kLog2Pi + log(v)) + quarter_sum(sm, c) / v);
    }
    return l;
  } else {
    const int p = M.p, q = M.q;
    if (k < p) {
      const double w = logistic_fn(qk);
      return 4.0 * log(w) + 4.0 * log1p(-w) + M.c_lbeta55 + log(w) + log1p(-w);
    }
    if (k <= p + q) return -0.5 * (kLog2Pi + qk * qk);
    const double sigma = exp(qk);
    const double v = sigma * sigma;
    return M.c_lhn1 - v / 2.0 + qk - 0.5 * (sm.ntr[c] * (kLog2Pi + log(v)) + quarter_sum(sm, c) / v);
  }
}

// ------------------------------------------------------------------ TMA ring
// Tile g of the kernel's sequence goes to slot g % kStages. The first kStages tiles of a pass are
// issued by thread 0 (every warp is past the previous pass's closing __syncthreads, so the slots
// are free); tile g + kStages is issued by the last warp to release tile g (counted in rel[]), so
// no thread ever blocks on a slot and the refill starts the moment the slot frees.
template <int KP>
__device__ __forceinline__ void issue_tile(Smem<KP>& sm, const ModelDev& M, int t, uint32_t g) {
  using G = Geom<KP>;
  const int slot = g % kStages;
  fence_proxy_async();  // generic-proxy reads of the slot before the async-proxy refill
  mbar_expect_tx(&sm.full[slot], G::TILE_BYTES);
  bulk_g2s(sm.xs[slot], M.xr + static_cast<size_t>(t) * G::TM * KP, G::TM * KP * 8, &sm.full[slot]);
  bulk_g2s(sm.ys[slot], M.y + static_cast<size_t>(t) * G::TM, G::TM * 8, &sm.full[slot]);
  bulk_g2s(sm.ks[slot], M.key + static_cast<size_t>(t) * G::TM, G::TM * 4, &sm.full[slot]);
}

#ifdef PCVG_GLM_TRACE
// Timeline probe (tools only): clock64 stamps of CTA 0, thread 0 for the passes of its first
// transition, printed at the end of the launch.
__device__ long long g_gtrace[64][14];
__device__ int g_gpass;
__device__ unsigned long long g_rtrace[16][8][14];  // CTAs 0..15, passes 32..39, globaltimer ns
__device__ int g_bpass[16];
__device__ unsigned long long g_ttrace[4][6];  // CTA 0, transitions 1..4: phase stamps (globaltimer)
#define TTRACE(i)                                                                                \
  do {                                                                                           \
    if (blockIdx.x == 0 && threadIdx.x == 0 && it >= 1 && it <= 4) g_ttrace[it - 1][(i)] = gtimer(); \
  } while (0)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define GTRACE(i)                                                                          \
  do {                                                                                     \
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_gpass < 64) g_gtrace[g_gpass][(i)] = clock64(); \
    if (blockIdx.x < 16 && threadIdx.x == 0 && g_bpass[blockIdx.x] >= 8 && g_bpass[blockIdx.x] < 16) \
      g_rtrace[blockIdx.x][g_bpass[blockIdx.x] - 8][(i)] = gtimer();                      \
  } while (0)
#else
#define GTRACE(i) \
  do {            \
  } while (0)
#define TTRACE(i) \
  do {            \
  } while (0)
#endif

// log(1 + e) for e in [0, 1] (the value pass's log1p(e^-|x|)) in ~11 FP64 operations instead of
// libm's ~40: d = 1 + e = c_j (1 + f) with c_j the centre of d's 1/64 interval (64-entry tables of
// 1 / c_j and log c_j), |f| <= 1/128, and log1p(f) by its degree-8 Taylor polynomial (truncation
// < 1e-19); below 1/128 the argument itself is f (c = 1), so small e keep full relative accuracy.
// Error ~2e-16 absolute per term, against the 1e-12 * sum|terms| parity budget of the log joint.
__device__ __forceinline__ double log1p_01(double e, const double* rc, const double* lc) {
  const bool small = e < 0.0078125;
  const double d = 1.0 + e;
  const int j = min(63, static_cast<int>((d - 1.0) * 64.0));
  const double f = small ? e : fma(d, rc[j], -1.0);
  double p = fma(f, -1.0 / 8.0, 1.0 / 7.0);
  p = fma(p, f, -1.0 / 6.0);
  p = fma(p, f, 1.0 / 5.0);
  p = fma(p, f, -1.0 / 4.0);
  p = fma(p, f, 1.0 / 3.0);
  p = fma(p, f, -0.5);
  p = fma(p, f * f, f);
  return small ? p : lc[j] + p;
}

// One pass over all observations for the 64 chains with weights sm.ws: G = X^T R into sm.rs as
// [col][chain]; the per-chain residual statistic (logistic: log-likelihood when VALUE; Gaussian:
// sum of squared training residuals, every pass) into sm.llp[quarter][chain].
template <int FAM, int KP, bool VALUE>
__device__ void grad_pass(Smem<KP>& sm, const ModelDev& M, uint32_t& gtile, int t0, int t1) {
  using G = Geom<KP>;
  constexpr bool kGauss = FAM != kLogistic;
  const int tid = threadIdx.x;
  const int w = tid >> 5, l = tid & 31;
  const int cg = w & 3, rq = w >> 2;
  const int ntiles = t1 - t0;
  const uint32_t g0 = gtile;
  if (tid == 0)
    for (int t = 0; t < kStages && t < ntiles; ++t) issue_tile(sm, M, t0 + t, g0 + t);
  int lo[2][2], hi[2][2];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int ch = 16 * cg + 8 * j + 2 * (l & 3) + e;
      lo[j][e] = sm.lo[ch];
      hi[j][e] = sm.hi[ch];
    }
  const double* wcol = sm.ws + 16 * cg + (l >> 2);
  // B fragments of X . W for this warp's 16 chains, held across the pass (WREG) or read per chunk
  double wf[G::WREG ? G::KS : 1][2];
  if constexpr (G::WREG) {
#pragma unroll
    for (int ks = 0; ks < G::KS; ++ks)
#pragma unroll
      for (int j = 0; j < 2; ++j) wf[ks][j] = wcol[(4 * ks + (l & 3)) * kLdS + 8 * j];
  }
  double gacc[G::PT][2][2];
#pragma unroll
  for (int pt = 0; pt < G::PT; ++pt)
#pragma unroll
    for (int j = 0; j < 2; ++j) gacc[pt][j][0] = gacc[pt][j][1] = 0.0;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  double* rblk = sm.rs + (16 * rq) * kLdS + 16 * cg;  // this warp's private 16 x 16 R block

  for (int tl = 0; tl < ntiles; ++tl) {
    const int t = t0 + tl;
    const uint32_t g = g0 + tl;
    const int slot = g % kStages;
    mbar_wait(&sm.full[slot], (g / kStages) & 1u);
    const double* xs = sm.xs[slot];
#pragma unroll 1
    for (int ch = 0; ch < G::CHUNKS; ++ch) {
      const int row0 = rq * G::ROWS_W + 16 * ch;
      double eta[2][2][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int j = 0; j < 2; ++j) eta[mt][j][0] = eta[mt][j][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < G::KS; ++ks) {
        double b[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = G::WREG ? wf[G::WREG ? ks : 0][j] : wcol[(4 * ks + (l & 3)) * kLdS + 8 * j];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const double a = xs[(row0 + 8 * mt + (l >> 2)) * KP + 4 * ks + (l & 3)];
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma(eta[mt][j][0], eta[mt][j][1], a, b[j]);
        }
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int row = row0 + 8 * mt + (l >> 2);
        const bool valid = t * G::TM + row < M.n;
        const double yv = sm.ys[slot][row];
        const int kv = sm.ks[slot][row];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          double r2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double x = eta[mt][j][e];
            const bool train = valid && static_cast<unsigned>(kv - lo[j][e]) >=
                                            static_cast<unsigned>(hi[j][e] - lo[j][e]);
            if constexpr (!kGauss && !VALUE) {
              const double rr = logistic_resid_fast(x, yv, yv - 1.0, sm.exp_hi32, sm.exp_lo32);  // no branch
              r2[e] = train ? rr : 0.0;
            } else if constexpr (!kGauss) {
              const double ex = exp_neg(fabs(x), sm.exp_tab);
              const double inv = rcp_1_2(1.0 + ex);
              const double sig = x >= 0.0 ? inv : ex * inv;
              r2[e] = train ? yv - sig : 0.0;
              if (train) acc[j][e] += yv * x - (fmax(x, 0.0) + log1p_01(ex, sm.l1p_rc, sm.l1p_lc));
              else if (valid && !isfinite(x)) acc[j][e] = CUDART_NAN;  // 0 * non-finite test term
            } else {
              const double r = yv - x;
              r2[e] = train ? r : 0.0;
              acc[j][e] = fma(r2[e], r, acc[j][e]);
              if (VALUE && valid && !train && !isfinite(r)) acc[j][e] = CUDART_NAN;
            }
          }
          *reinterpret_cast<double2*>(&rblk[(8 * mt + (l >> 2)) * kLdS + 8 * j + 2 * (l & 3)]) =
              make_double2(r2[0], r2[1]);
        }
      }
      __syncwarp();
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int m = 4 * ks + (l & 3);
        double b[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = rblk[m * kLdS + 8 * j + (l >> 2)];
#pragma unroll
        for (int pt = 0; pt < G::PT; ++pt) {
          const double a = xs[(row0 + m) * KP + 8 * pt + (l >> 2)];
#pragma unroll
          for (int j = 0; j < 2; ++j) dmma(gacc[pt][j][0], gacc[pt][j][1], a, b[j]);
        }
      }
      __syncwarp();
    }
    if (l == 0 && tl + kStages < ntiles) {
      const unsigned int old = atomicAdd(&sm.rel[slot], 1u);
      if ((old + 1u) % G::WARPS == 0u) issue_tile(sm, M, t + kStages, g + kStages);
    } else if (l == 0) {
      atomicAdd(&sm.rel[slot], 1u);
    }
  }
  gtile = g0 + ntiles;
  GTRACE(1);
  __syncthreads();
  GTRACE(11);
  // Stage G [col][chain] into sm.rs: every row group stores its partial at once - row group 0 into
  // sm.rs, groups 1..3 into the idle TMA ring slots ([col][64], 16-byte granules XOR-swizzled by
  // col so a warp's 8 columns hit distinct banks) - then all threads add the four in a fixed tree,
  // (g0 + g1) + (g2 + g3): two barriers instead of four sequential rounds.
  static_assert(G::RQ == 4, "four row groups");
  static_assert(G::TM * KP + G::XPAD >= KP * kC, "a ring slot holds one G partial");
  auto part_idx = [](int p, int ch) { return p * kC + (((ch >> 1) ^ ((p & 7) << 1)) << 1) + (ch & 1); };
#pragma unroll
  for (int pt = 0; pt < G::PT; ++pt) {
    const int p = 8 * pt + (l >> 2);
    if (p < KP) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int ch = 16 * cg + 8 * j + 2 * (l & 3);
        double2* dst = rq == 0 ? reinterpret_cast<double2*>(&sm.rs[p * kLdS + ch])
                               : reinterpret_cast<double2*>(&sm.xs[rq - 1][part_idx(p, ch)]);
        *dst = make_double2(gacc[pt][j][0], gacc[pt][j][1]);
      }
    }
  }
  if (VALUE || kGauss) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = acc[j][e];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (l < 4) sm.llp[rq][16 * cg + 8 * j + 2 * l + e] = v;
      }
  }
  __syncthreads();
  for (int i = tid; i < KP * kC; i += G::THREADS) {
    const int p = i / kC, ch = i % kC, x = part_idx(p, ch);
    double* d = &sm.rs[p * kLdS + ch];
    *d = (*d + sm.xs[0][x]) + (sm.xs[1][x] + sm.xs[2][x]);
  }
  __syncthreads();
}

// Sums the staged partials (G in sm.rs rows 0..KP-1, residual statistic in sm.llp) over the CS CTAs
// of the cluster and the NC clusters of the chain tile, in place: afterwards sm.rs rows 0..KP hold
// the reduced G and (row KP) the residual statistic, identical bits in every CTA of the tile.
//  * CS = 1: the staged rows already are the sums (row KP = the row-group sum).
//  * CS > 1, push-based over DSMEM: rank o owns rows [o*per, (o+1)*per). Every rank bulk-copies
//    (cp.async.bulk shared::cta -> shared::cluster, SASS UBLKCP) each owner's rows of its partial
//    into the owner's receive slot (sm.gt) completing on the owner's mbarrier; the owner adds the
//    CS partials in rank order, then bulk-copies its reduced rows into every other rank's sm.rs.
//    Two mbarrier waits per pass and no cluster barrier (round 1 pulled the partials with DSMEM
//    loads between three cluster.sync: ~6 us of a ~31 us cfg2 K-fold pass, ~2 us now).
//  * NC > 1 (reduce_clusters): between the two steps, each owner's rows meet the same rows of the
//    other clusters in global memory (published by pass parity, one arrival counter per tile and
//    rank) and are added in cluster order.
// Hazards are ordered by the data flow: a rank's partial rows are overwritten (gather) only after
// their owner received them; an owner's receive slot is rewritten (next pass) only after its
// gather reached the sender; the mbarriers are armed (expect_tx) once per pass by thread 0 and
// may see bytes before they are armed (the transaction count goes negative, the phase waits for
// the local arrival). The launch syncs the cluster once after the barriers are initialised.
template <int KP>
__device__ void reduce_clusters(Smem<KP>& sm, const ModelDev& M, int tile, int nc, int clus, int crank, int r0,
                                int r1, uint32_t& gpass) {
  using G = Geom<KP>;
  constexpr int kThreads = G::THREADS;
  constexpr int kE = G::RROWS * kC;
  const int tid = threadIdx.x;
  const uint32_t par = gpass & 1u;
  ++gpass;
  if (r1 <= r0) return;  // no rows: neither does this rank in any other cluster
  double* base = M.glm_part + (static_cast<size_t>(tile) * 2 + par) * nc * kE;
  const int n = (r1 - r0) * kC;
  GTRACE(5);
  for (int i = tid; i < n; i += kThreads) {
    const int row = r0 + i / kC, c = i % kC;
    __stcg(base + static_cast<size_t>(clus) * kE + row * kC + c, sm.rs[row * kLdS + c]);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    cuda::atomic_ref<unsigned int, cuda::thread_scope_device> cnt(M.glm_cnt[tile * 16 + crank]);
    cnt.fetch_add(1u, cuda::memory_order_release);
    const unsigned int target = (gpass) * static_cast<unsigned int>(nc);
    while (cnt.load(cuda::memory_order_acquire) < target) __nanosleep(32);
  }
  __syncthreads();
  GTRACE(6);
  // every partial of an element loaded before any is added, then summed in cluster order
  constexpr int kBatch = 8;  // loads in flight per batch (nc <= kMaxClusters = 16: two batches)
  for (int i = tid; i < n; i += kThreads) {
    const int row = r0 + i / kC, c = i % kC;
    double x = 0.0;
    for (int q0 = 0; q0 < nc; q0 += kBatch) {
      double v[kBatch];
#pragma unroll
      for (int q = 0; q < kBatch; ++q)
        v[q] = q0 + q < nc ? __ldcg(base + static_cast<size_t>(q0 + q) * kE + row * kC + c) : 0.0;
#pragma unroll
      for (int q = 0; q < kBatch; ++q)
        if (q0 + q < nc) x = q0 + q == 0 ? v[q] : x + v[q];
    }
    sm.rs[row * kLdS + c] = x;
  }
}

template <int KP>
__device__ void reduce_pass(Smem<KP>& sm, int cs, const ModelDev& M, int tile, int nc, int clus, int crank,
                            uint32_t& gpass, uint32_t& cpass) {
  using G = Geom<KP>;
  constexpr int kThreads = G::THREADS;
  constexpr int R = G::RROWS;
  constexpr uint32_t kRowBytes = kLdS * sizeof(double);
  const int tid = threadIdx.x;
  if (tid < kC) sm.rs[KP * kLdS + tid] = rq_sum<G::RQ>(sm.llp, tid);
  if (cs == 1) {
    __syncthreads();
    if (nc > 1) {
      reduce_clusters(sm, M, tile, nc, clus, 0, 0, R, gpass);
      __syncthreads();
    }
    return;
  }
  const int me = crank;
  const int per = (R + cs - 1) / cs;
  const int r0 = min(R, me * per), r1 = min(R, r0 + per);
  const uint32_t ph = cpass & 1u;
  ++cpass;
  tc::fence_proxy_async();  // the staged rows are read by the bulk copies
  __syncthreads();
  GTRACE(7);
  if (tid == 0) {
    tc::mbar_expect_tx(&sm.rbar[0], static_cast<uint32_t>(cs - 1) * (r1 - r0) * kRowBytes);
    tc::mbar_expect_tx(&sm.rbar[1], static_cast<uint32_t>(R - (r1 - r0)) * kRowBytes);
    for (int j = 1; j < cs; ++j) {
      const int o = (me + j) % cs;  // owners in a rotated order: not every rank hits rank 0 first
      const int a = min(R, o * per), b = min(R, a + per);
      if (b <= a) continue;
      const int slot = me < o ? me : me - 1;
      tc::bulk_s2c(tc::cluster_addr(&sm.gt[slot * per * kLdS], o), &sm.rs[a * kLdS],
                   static_cast<uint32_t>(b - a) * kRowBytes, tc::cluster_addr(&sm.rbar[0], o));
    }
  }
  if (r1 > r0) {
    tc::mbar_wait(&sm.rbar[0], ph);
    for (int i = tid; i < (r1 - r0) * kC; i += kThreads) {
      const int rr = i / kC, c = i % kC, row = r0 + rr;
      double x = 0.0;
      for (int q = 0; q < cs; ++q) {
        const double v = q == me ? sm.rs[row * kLdS + c] : sm.gt[((q < me ? q : q - 1) * per + rr) * kLdS + c];
        x = q == 0 ? v : x + v;
      }
      sm.rs[row * kLdS + c] = x;
    }
  }
  GTRACE(8);
  if (nc > 1) {
    __syncthreads();
    reduce_clusters(sm, M, tile, nc, clus, crank, r0, r1, gpass);
  }
  tc::fence_proxy_async();  // the reduced rows are read by the bulk copies
  __syncthreads();
  GTRACE(9);
  if (tid == 0 && r1 > r0) {
    for (int j = 1; j < cs; ++j) {
      const int o = (me + j) % cs;
      tc::bulk_s2c(tc::cluster_addr(&sm.rs[r0 * kLdS], o), &sm.rs[r0 * kLdS],
                   static_cast<uint32_t>(r1 - r0) * kRowBytes, tc::cluster_addr(&sm.rbar[1], o));
    }
  }
  tc::mbar_wait(&sm.rbar[1], ph);
  GTRACE(10);
}

// HS / DSS state of one chain after hmc_step + log_pred (engine.cpp:360-373; warm-up
// hmc.cpp:133-145), run by the chain thread over the fold's test rows in order: pred_derivs /
// pred_sample of grouped_regression.cpp:190-213 (J = 1) and seasonal_ar.cpp:133-150. Every rank
// of a cluster draws the DSS normals (identical stream state); only the writer rank stores.
template <int FAM, int KP>
__device__ void glm_score_extra(const ModelDev& M, const ChainsDev& S, int gc, int fold,
                                const double* pos, bool warm, bool writer, ChainRng& R) {
  const ExtraDev& X = S.X;
  const int nch = S.nch, L = S.L, kf = fold - S.fold0, cl = gc % L;
  double vy, sy;
  if constexpr (FAM == kGrouped) {
    sy = exp(pos[static_cast<size_t>(M.nc + 3) * nch]);
    vy = sy * sy;
  } else {
    const double u = pos[static_cast<size_t>(M.p + M.q + 1) * nch];
    vy = exp(2.0 * u);
    sy = exp(u);
  }
  const int s0 = M.fold_seg[fold], s1 = M.fold_seg[fold + 1];
  int rt = 0;
  for (int s = s0; s < s1; ++s) {
    for (int tt = M.seg_row[s]; tt < M.seg_row[s + 1]; ++tt, ++rt) {
      const double z = X.kind == 2 ? R.normal() : 0.0;
      if (!writer) continue;
      const int i = M.seg_rows[tt];
      const double* xrow = M.xr + static_cast<size_t>(i) * KP;
      double mean = 0.0;
      for (int k = 0; k < M.dim; ++k) {
        const int col = col_of<FAM>(M, k);
        if (col >= 0) mean = fma(xrow[col], w_of<FAM>(M, k, pos[static_cast<size_t>(k) * nch]), mean);
      }
      if (X.kind == 1) extra_hs_row(X, kf, cl, L, rt, -(M.y[i] - mean) / vy, -1.0 / vy, warm);
      else extra_dss_row(X, kf, cl, L, rt, mean + sy * z, warm);
    }
  }
  if (X.kind == 2 && !warm && writer) extra_dss_cov(X, kf, cl, L, 0, 1);
}

template <int FAM, int KP>
__global__ void __launch_bounds__(Geom<KP>::THREADS, 1) glm_kernel(ModelDev M, ChainsDev S, RunArgs A, int cs,
                                                           int tile0, int nc) {
  using G = Geom<KP>;
  constexpr int kThreads = G::THREADS, kOwners = G::OWNERS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem<KP>& sm = *reinterpret_cast<Smem<KP>*>(smem_raw);
  const int tid = threadIdx.x;
  const int nch = S.nch;
  const int dim = M.dim;
  const size_t plane = static_cast<size_t>(dim) * nch;
  const int span = cs * nc;                                     // CTAs per chain tile
  const int tile = tile0 + blockIdx.x / span, gr = blockIdx.x % span;  // chain tile, rank in the tile
  const int clus = gr / cs, crank = gr % cs;                   // cluster of the tile, rank in the cluster
  const bool writer = gr == 0;                                 // rank 0 owns the final global writes
  const int ntiles_all = (M.n + G::TM - 1) / G::TM;
  const int t0 = gr * ntiles_all / span, t1 = (gr + 1) * ntiles_all / span;
  uint32_t gpass = 0;                                          // second-level reductions done
  uint32_t cpass = 0;                                          // cluster reductions done
  const int oc = tid & (kC - 1), ok = tid / kC;  // owner: chain oc, params ok + 8j
  const int ogc = tile * kC + oc;
  const bool ovalid = ogc < nch;
  const bool is_chain = tid < kC;
  const int gc = tile * kC + tid;
  const bool cvalid = is_chain && gc < nch;

  if (tid < kStages) {
    mbar_init(&sm.full[tid], 1);
    sm.rel[tid] = 0u;
  }
  if (tid < 2) mbar_init(&sm.rbar[tid], 1);
  if (tid < 16) sm.exp_tab[tid] = exp2(-tid / 16.0);
  if (tid < 64) {
    const double cj = 1.0 + (tid + 0.5) / 64.0;
    sm.l1p_rc[tid] = 1.0 / cj;
    sm.l1p_lc[tid] = log(cj);
  }
  if (tid < 32) {
    const double v = exp2(-tid / 32.0);
    sm.exp_hi32[tid] = __double2hiint(v);
    sm.exp_lo32[tid] = __double2loint(v);
  }
  for (int i = tid; i < KP * kLdS; i += kThreads) sm.ws[i] = 0.0;
  for (int i = tid; i < dim; i += kThreads) sm.im[i] = __ldg(M.inv_mass + i);
  fence_mbar_init();
  uint32_t gtile = 0;

  ChainRng R;
  double lp0 = 0.0, warm = 0.0;
  int64_t div_count = 0;
  int fold = M.K;
  if (is_chain) {
    if (cvalid) {
      fold = S.fold_override ? S.fold_override[gc] : S.fold0 + gc / S.L;
      sm.lo[tid] = M.fold_lo[fold];
      sm.hi[tid] = M.fold_hi[fold];
      sm.ntr[tid] = M.n_train[fold];
      sm.cur[tid] = S.cur[gc];
      sm.fold[tid] = fold;
      lp0 = S.lp0[gc];
      R.init(S.seed, S.rng_stream[gc], S.rng_pos[gc], S.rng_cached[gc], S.rng_has[gc] != 0);
    } else {
      sm.lo[tid] = 0;
      sm.hi[tid] = 0;
      sm.ntr[tid] = M.n;
      sm.cur[tid] = 0;
      sm.fold[tid] = M.K;
    }
  }
  __syncthreads();
  if (cs > 1) cooperative_groups::this_cluster().sync();  // reduction barriers initialised cluster-wide

  // owners: publish parameters + GEMM weights of their slots
  auto put_q = [&](int k, double q) {
    sm.qs[k * kLdS + oc] = q;
    const int col = col_of<FAM>(M, k);
    if (col >= 0) sm.ws[col * kLdS + oc] = w_of<FAM>(M, k, q);
  };
  auto lp_from_partials = [&](int c) {
    double pr = 0.0;
#pragma unroll
    for (int o = 0; o < kOwners; ++o) pr += sm.pri[o][c];
    if constexpr (FAM == kLogistic) return quarter_sum(sm, c) + pr;
    else return pr;
  };

  if (A.mode == kModeEval) {
    {
      const int cu = sm.cur[oc];
#pragma unroll
      for (int j = 0; j < G::OWN; ++j) {
        const int k = ok + kOwners * j;
        if (k < dim) put_q(k, ovalid ? S.pos[cu * plane + static_cast<size_t>(k) * nch + ogc] : 0.0);
      }
    }
    __syncthreads();
    grad_pass<FAM, KP, true>(sm, M, gtile, t0, t1);
    reduce_pass(sm, cs, M, tile, nc, clus, crank, gpass, cpass);
    double pr = 0.0;
    const int cu = sm.cur[oc];
#pragma unroll
    for (int j = 0; j < G::OWN; ++j) {
      const int k = ok + kOwners * j;
      if (k < dim) {
        const double q = sm.qs[k * kLdS + oc];
        const int col = col_of<FAM>(M, k);
        const double gk = col >= 0 ? sm.rs[col * kLdS + oc] : 0.0;
        if (ovalid && writer) S.grad[cu * plane + static_cast<size_t>(k) * nch + ogc] = grad_of<FAM, KP>(M, sm, k, oc, gk, q);
        pr += logp_of<FAM, KP>(M, sm, k, oc, q);
      }
    }
    sm.pri[ok][oc] = pr;
    __syncthreads();
    if (cvalid && writer) {
      const double lp = lp_from_partials(tid);
      S.lp0[gc] = lp;
      if (A.out_a) A.out_a[gc] = lp;
    }
    // rank 0 may still be reading the other ranks' reduced slices (reduce_pass copy phase): no
    // rank may exit (releasing its shared memory) before every rank is past that point
    if (cs > 1) cooperative_groups::this_cluster().sync();
    return;
  }

  const double eps = M.step, half = 0.5 * M.step;
  const int n_lf = M.n_lf;
  for (int64_t it = 0; it < A.n_iters; ++it) {
    TTRACE(0);
    if (A.mode != kModePred) {
      // -- momentum refresh (reference draw order) -> staging in sm.rs. The Box-Muller pairs of a
      //    chain sit at known positions of its stream, so its 8 owner threads draw them in parallel
      //    (normal_pair_at, the same bits as R.normal()); the chain thread then advances its stream
      //    past them and sums the kinetic energy in dimension order.
      double k0 = 0.0;
      if (A.mode == kModeProbe) {
        if (is_chain) {
          for (int k = 0; k < dim; ++k) {
            const double mk = sm.im[k];
            const double p = cvalid ? A.probe_momentum[static_cast<size_t>(gc) * dim + k] : 0.0;
            k0 += mk * p * p;
            sm.rs[k * kLdS + tid] = p;
          }
        }
      } else {
        if (is_chain) {
          sm.rng_pos[tid] = R.pos;
          sm.rng_has[tid] = R.has_cached ? 1 : 0;
          sm.rng_cached[tid] = R.cached;
        }
        __syncthreads();
        if (ovalid) {
          const int h = sm.rng_has[oc];
          const uint64_t pos0 = sm.rng_pos[oc];
          const int npairs = (dim - h + 1) / 2;
          if (ok == 0 && h) sm.rs[oc] = sm.rng_cached[oc] / sqrt(sm.im[0]);
          const uint64_t stream = S.rng_stream[ogc];
          for (int j = ok; j < npairs; j += kOwners) {
            double a, b;
            normal_pair_at(static_cast<uint32_t>(S.seed), static_cast<uint32_t>(S.seed >> 32), stream,
                           pos0 + 4ull * j, &a, &b);
            const int k = h + 2 * j;
            sm.rs[k * kLdS + oc] = a / sqrt(sm.im[k]);
            if (k + 1 < dim) sm.rs[(k + 1) * kLdS + oc] = b / sqrt(sm.im[k + 1]);
            else sm.rng_tail[oc] = b;  // odd count: the pair's second value stays cached
          }
        }
        __syncthreads();
        if (cvalid) {
          const int h = R.has_cached ? 1 : 0;
          const int npairs = (dim - h + 1) / 2;
          R.pos += 4ull * npairs;
          R.buf_block = ~0ull;
          R.has_cached = ((dim - h) & 1) != 0;
          if (R.has_cached) R.cached = sm.rng_tail[tid];
          for (int k = 0; k < dim; ++k) {
            const double mk = sm.im[k];
            const double p = sm.rs[k * kLdS + tid];
            k0 += mk * p * p;
          }
        }
      }
      if (is_chain) sm.bad[tid] = 0;
      __syncthreads();
      // -- half kick + first drift (owners)
      double pown[G::OWN];
      {
        const int cu = sm.cur[oc];
        bool bad = false;
#pragma unroll
        for (int j = 0; j < G::OWN; ++j) {
          const int k = ok + kOwners * j;
          double q = 0.0, p = 0.0;
          if (k < dim) {
            if (ovalid) {
              const size_t gi = cu * plane + static_cast<size_t>(k) * nch + ogc;
              p = sm.rs[k * kLdS + oc] + half * S.grad[gi];
              q = S.pos[gi] + eps * sm.im[k] * p;
              bad |= !isfinite(q);
            }
            put_q(k, q);
          }
          pown[j] = p;
        }
        if (bad) sm.bad[oc] = 1;
      }
      __syncthreads();
      TTRACE(1);
      // -- leapfrog: n_lf gradient passes
      for (int s = 0; s < n_lf; ++s) {
        const bool last = s == n_lf - 1;
        GTRACE(0);
        if (last) grad_pass<FAM, KP, true>(sm, M, gtile, t0, t1);
        else grad_pass<FAM, KP, false>(sm, M, gtile, t0, t1);
        GTRACE(2);
        reduce_pass(sm, cs, M, tile, nc, clus, crank, gpass, cpass);
        GTRACE(3);
        const double scale = last ? half : eps;
        const int cu = sm.cur[oc];
        bool bad = false;
        double part = 0.0, part2 = 0.0;
        double gk_new[G::OWN];
#pragma unroll
        for (int j = 0; j < G::OWN; ++j) {
          const int k = ok + kOwners * j;
          gk_new[j] = 0.0;
          if (k < dim) {
            const double q = sm.qs[k * kLdS + oc];
            const int col = col_of<FAM>(M, k);
            const double g = grad_of<FAM, KP>(M, sm, k, oc, col >= 0 ? sm.rs[col * kLdS + oc] : 0.0, q);
            gk_new[j] = g;
            bad |= !isfinite(g);
            pown[j] += scale * g;
            bad |= !isfinite(pown[j]);
            if (last) {
              part += sm.im[k] * pown[j] * pown[j];
              part2 += logp_of<FAM, KP>(M, sm, k, oc, q);
              // the proposal plane: rank 0 of a cluster (its ranks sync on the cluster barrier); over
              // several clusters every CTA stores the same bits and reads back its own stores
              if (ovalid && (writer || nc > 1)) {
                const size_t gi = (cu ^ 1) * plane + static_cast<size_t>(k) * nch + ogc;
                S.pos[gi] = q;
                S.grad[gi] = g;
              }
              if (ovalid && writer && A.mode == kModeProbe && A.traj) A.traj[static_cast<size_t>(ogc) * dim + k] = pown[j];
            }
          }
        }
        (void)gk_new;
        GTRACE(12);
        __syncthreads();  // every owner read G / q / llp before they change
        GTRACE(13);
        if (!last) {
#pragma unroll
          for (int j = 0; j < G::OWN; ++j) {
            const int k = ok + kOwners * j;
            if (k < dim) {
              const double q = sm.qs[k * kLdS + oc] + eps * sm.im[k] * pown[j];
              bad |= !isfinite(q);
              put_q(k, q);
            }
          }
        } else {
          sm.red[ok][oc] = part;
          sm.pri[ok][oc] = part2;
        }
        if (bad) sm.bad[oc] = 1;
        __syncthreads();
        GTRACE(4);
#ifdef PCVG_GLM_TRACE
        if (blockIdx.x == 0 && threadIdx.x == 0) ++g_gpass;
        if (blockIdx.x < 16 && threadIdx.x == 0) ++g_bpass[blockIdx.x];
#endif
      }
      TTRACE(2);
      // -- energies, Metropolis (chain thread)
      if (is_chain) {
        double k1 = 0.0;
#pragma unroll
        for (int o = 0; o < kOwners; ++o) k1 += sm.red[o][tid];
        const double lp1 = lp_from_partials(tid);
        const bool bad = sm.bad[tid] != 0 || sm.fold[tid] == M.broken_fold;
        const double h0 = -lp0 + 0.5 * k0;
        const double h1 = bad ? CUDART_NAN : -lp1 + 0.5 * k1;
        const double dh = h1 - h0;
        const bool divergent = bad || isnan(dh) || (isfinite(dh) && fabs(dh) > 1000.0);
        bool accepted = false;
        if (divergent) {
          ++div_count;
        } else {
          const double u = A.mode == kModeProbe ? (cvalid ? A.probe_u[gc] : 0.5) : R.uniform();
          if (log(u) < -dh) {
            accepted = true;
            sm.cur[tid] ^= 1;
            lp0 = lp1;
          }
        }
        if (cvalid && writer && A.mode == kModeProbe) {
          A.out_a[gc] = h0;
          A.out_b[gc] = h1;
          A.out_flags[gc] = (accepted ? 1 : 0) | (divergent ? 2 : 0);
        }
        if (cvalid && writer && A.mode == kModeChain) {  // trace row (it, chain) = it * nch + gc
          const size_t row = static_cast<size_t>(it) * nch + gc;
          if (A.traj_div) A.traj_div[row] = (accepted ? 1 : 0) | (divergent ? 2 : 0);
          if (A.out_a) A.out_a[row] = h0;
          if (A.out_b) A.out_b[row] = h1;
        }
      }
      // rank 0's proposal writes must be visible to the cluster before the next half kick
      if (cs > 1) cooperative_groups::this_cluster().sync();
      else __syncthreads();
      if (A.mode == kModeProbe) continue;
      if (A.mode == kModeChain) {
        const int cu = sm.cur[oc];
        if (ovalid && writer) {
#pragma unroll
          for (int j = 0; j < G::OWN; ++j) {
            const int k = ok + kOwners * j;
            if (k < dim && A.traj)
              A.traj[(static_cast<size_t>(it) * nch + ogc) * dim + k] = S.pos[cu * plane + static_cast<size_t>(k) * nch + ogc];
          }
        }
        continue;
      }
    }
    TTRACE(3);
    // -- log_pred at the current position: the cs ranks of the tile's first cluster and the 8 owner
    //    threads of a chain split its fold's test rows (K-fold: 1,000 rows at cfg2; row tt goes to
    //    rank (tt / 8) % cs, owner tt % 8) with the position staged [k][chain] in sm.rs; each rank
    //    adds its owner partials in owner order, rank 0's chain thread adds the rank partials in
    //    rank order (DSMEM) and updates the accumulators
    const bool lp_rank = clus == 0;
    if (lp_rank) {
      const int cu = sm.cur[oc];
#pragma unroll
      for (int j = 0; j < G::OWN; ++j) {
        const int k = ok + kOwners * j;
        if (k < dim) sm.rs[k * kLdS + oc] = ovalid ? S.pos[cu * plane + static_cast<size_t>(k) * nch + ogc] : 0.0;
      }
    }
    __syncthreads();
    {
      double part = 0.0;
      const int ofold = sm.fold[oc];
      if (lp_rank && ovalid && ofold < M.K) {
        const double* th = sm.rs + oc;
        double v_pred = 1.0;
        if constexpr (FAM == kGrouped) {
          const double sy = exp(th[(M.nc + 3) * kLdS]);
          v_pred = sy * sy;  // grouped_regression.cpp:240-241
        } else if constexpr (FAM == kSeasonal) {
          v_pred = exp(2.0 * th[(M.p + M.q + 1) * kLdS]);  // seasonal_ar.cpp:110
        }
        const int s0 = M.fold_seg[ofold], s1 = M.fold_seg[ofold + 1];
        const int r0 = M.seg_row[s0], r1 = M.seg_row[s1];  // the fold's test rows, contiguous
        for (int tt = r0 + crank * kOwners + ok; tt < r1; tt += kOwners * cs) {
          const int i = M.seg_rows[tt];
          const double* xrow = M.xr + static_cast<size_t>(i) * KP;
          double eta = 0.0;
          if constexpr (FAM == kLogistic) {
            // the padded row as KP / 2 independent 16-byte loads and four partial sums (column k
            // of X is parameter k; padding columns are zero and get weight 0): a row's loads are
            // in flight together instead of one dependent load + FMA per column (K-fold cfg2:
            // 1,000 test rows per fold made log_pred ~1/3 of a transition)
            static_assert(KP % 4 == 0, "row pairs");
            const double2* x2 = reinterpret_cast<const double2*>(xrow);
            double e4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int kk = 0; kk < KP / 2; ++kk) {
              const double2 xv = __ldg(x2 + kk);
              const int k = 2 * kk;
              const double w0 = k < dim ? th[k * kLdS] : 0.0;
              const double w1 = k + 1 < dim ? th[(k + 1) * kLdS] : 0.0;
              e4[(2 * kk) & 3] = fma(xv.x, w0, e4[(2 * kk) & 3]);
              e4[(2 * kk + 1) & 3] = fma(xv.y, w1, e4[(2 * kk + 1) & 3]);
            }
            eta = (e4[0] + e4[1]) + (e4[2] + e4[3]);
            // log p(y | eta) = y eta - (max(eta, 0) + log1p(e^-|eta|)) with the value pass's exp / log1p
            part += M.y[i] * eta - (fmax(eta, 0.0) + log1p_01(exp_neg(fabs(eta), sm.exp_tab), sm.l1p_rc, sm.l1p_lc));
          } else {
            for (int k = 0; k < dim; ++k) {
              const int col = col_of<FAM>(M, k);
              if (col >= 0) eta = fma(xrow[col], w_of<FAM>(M, k, th[k * kLdS]), eta);
            }
            part += normal_logpdf(M.y[i], eta, v_pred);
          }
        }
      }
      sm.red[ok][oc] = part;
    }
    __syncthreads();
    double sp = 0.0;
    if (is_chain) {
#pragma unroll
      for (int o = 0; o < kOwners; ++o) sp += sm.red[o][tid];
    }
    if (cs > 1) {
      if (is_chain) sm.lpp[tid] = sp;
      cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
      cl.sync();  // every rank's partials published
      if (cvalid && writer) {
        sp = 0.0;
        for (int q = 0; q < cs; ++q) sp += cl.map_shared_rank(sm.lpp, q)[tid];
      }
      // no rank may exit while rank 0 still reads its partials (the next transition's syncs order
      // the reuse of sm.lpp otherwise)
      if (it + 1 == A.n_iters || A.mode == kModePred) cl.sync();
    }
    if (cvalid && writer) {
      if (A.mode == kModePred) {
        if (A.out_a) A.out_a[gc] = sp;
      } else if (A.mode == kModeWarmup) {
        warm += sp;
      } else {
        accum_observe(S.acc, gc, nch, sp, A.iter0 + it, A.planned_n, A.D, A.b);
      }
    }
    if constexpr (FAM != kLogistic) {
      if (cvalid && S.X.kind != 0 && fold < M.K && A.mode != kModePred)
        glm_score_extra<FAM, KP>(M, S, gc, fold, S.pos + sm.cur[tid] * plane + gc,
                                 A.mode == kModeWarmup, writer, R);
    }
    TTRACE(4);
    if (A.mode == kModePred) break;
  }
#ifdef PCVG_GLM_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0 && g_gpass >= 32 && g_gpass < 1000) {
    printf("pass: start tiles_done staged reduced owners_done | cluster-level-done arrived (cycles), cs=%d nc=%d\n",
           cs, nc);
    for (int p = 0; p < 32 && p < 64; ++p)
      printf("%2d: %lld %lld %lld %lld | %lld %lld | next start +%lld\n", p, g_gtrace[p][1] - g_gtrace[p][0],
             g_gtrace[p][2] - g_gtrace[p][0], g_gtrace[p][3] - g_gtrace[p][0], g_gtrace[p][4] - g_gtrace[p][0],
             g_gtrace[p][5] - g_gtrace[p][0], g_gtrace[p][6] - g_gtrace[p][0],
             p + 1 < 32 ? g_gtrace[p + 1][0] - g_gtrace[p][0] : 0LL);
    g_gpass = 1000;
    for (int t = 0; t < 3; ++t)
      printf("transition %d (ns from start): momentum+kick %lld | passes %lld | metropolis %lld | log_pred+accum %lld | next %lld\n", t + 1,
             (long long)(g_ttrace[t][1] - g_ttrace[t][0]), (long long)(g_ttrace[t][2] - g_ttrace[t][1]),
             (long long)(g_ttrace[t][3] - g_ttrace[t][2]), (long long)(g_ttrace[t][4] - g_ttrace[t][3]),
             (long long)(g_ttrace[t + 1][0] - g_ttrace[t][4]));
    printf("per-CTA (ns from CTA0 pass start): cta pass | tiles allwarps staged red-start rows-reduced pre-gather gathered glob-publish glob-arrived reduced own-done own-synced owners\n");
    for (int p = 0; p < 3; ++p) {
      const unsigned long long z = g_rtrace[0][p][0];
      for (int b = 0; b < 16; ++b)
        printf("%2d %d | %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld (start %lld)\n", b, p, (long long)(g_rtrace[b][p][1] - z),
               (long long)(g_rtrace[b][p][11] - z), (long long)(g_rtrace[b][p][2] - z), (long long)(g_rtrace[b][p][7] - z), (long long)(g_rtrace[b][p][8] - z),
               (long long)(g_rtrace[b][p][9] - z), (long long)(g_rtrace[b][p][10] - z), (long long)(g_rtrace[b][p][5] - z), (long long)(g_rtrace[b][p][6] - z),
               (long long)(g_rtrace[b][p][3] - z), (long long)(g_rtrace[b][p][12] - z), (long long)(g_rtrace[b][p][13] - z), (long long)(g_rtrace[b][p][4] - z), (long long)(g_rtrace[b][p][0] - z));
    }
  }
#endif
  if (cvalid && writer && A.mode != kModePred) {
    S.cur[gc] = static_cast<int8_t>(sm.cur[tid]);
    S.lp0[gc] = lp0;
    S.rng_pos[gc] = R.pos;
    S.rng_cached[gc] = R.cached;
    S.rng_has[gc] = R.has_cached ? 1 : 0;
    S.divergences[gc] += div_count;
    if (A.mode == kModeWarmup) S.warm_sum[gc] += warm;
  }
}

template <int FAM, int KP>
cudaError_t launch_t(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st) {
  const int tiles = (S.nch + kC - 1) / kC;
  if (tiles == 0) return cudaSuccess;
  {
    // 16-CTA clusters (non-portable) for the fewest-chain configurations (cfg2 K-fold: 80 chains)
    cudaError_t e = ensure_kernel_smem(reinterpret_cast<const void*>(glm_kernel<FAM, KP>), sizeof(Smem<KP>), true);
    if (e != cudaSuccess) return e;
  }
  auto launch = [&](int tile0, int ntiles, int cs, int nc) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles * cs * nc);
    cfg.blockDim = dim3(Geom<KP>::THREADS);
    cfg.dynamicSmemBytes = sizeof(Smem<KP>);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (cs > 1) {
      at[na].id = cudaLaunchAttributeClusterDimension;
      at[na].val.clusterDim.x = cs;
      at[na].val.clusterDim.y = 1;
      at[na].val.clusterDim.z = 1;
      ++na;
    }
    if (nc > 1) {  // co-residency of every CTA: the second-level reduction waits on the others
      at[na].id = cudaLaunchAttributeCooperative;
      at[na].val.cooperative = 1;
      ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    ++sampler_launch_count();
    return cudaLaunchKernelEx(&cfg, glm_kernel<FAM, KP>, M, S, A, cs, tile0, nc);
  };
  // Concurrently schedulable clusters of each size (a cluster must fit in one GPC): a 16-CTA cluster
  // only pays while every tile's cluster runs at once, else halve it.
  auto fits = [&](int c) {
    return cached_launch_fact(reinterpret_cast<const void*>(glm_kernel<FAM, KP>), c, [&] {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(c);
      q.blockDim = dim3(Geom<KP>::THREADS);
      q.dynamicSmemBytes = sizeof(Smem<KP>);
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = c;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, glm_kernel<FAM, KP>, &q) != cudaSuccess) nclusters = 0;
      cudaGetLastError();
      return nclusters;
    });
  };
  int cs = glm_cluster_size(M.n, KP, S.nch);
  while (cs > 8 && fits(cs) < tiles) cs /= 2;
  if (const char* e = std::getenv("PCVG_GLM_CS")) cs = std::atoi(e);  // tuning only
  // several clusters per tile: as many as the device can keep resident at once (the cooperative
  // launch requires it), for the cluster size that puts the most CTAs on each tile
  int nc = 1;
  const int cs_single = cs;
  const bool scratch = M.glm_part != nullptr && M.glm_cnt != nullptr;
  for (int c = cs; c >= 8 && cs >= 8; c /= 2) {
    const int k = std::min(glm_clusters_per_tile(M.n, KP, S.nch, c, scratch), fits(c) / tiles);
    if (k > 1 && c * k > cs * nc) {
      cs = c;
      nc = k;
    }
  }
  static const bool verbose = std::getenv("PCVG_VERBOSE") != nullptr;  // tuning only
  if (nc > 1) {
    // Two cooperative grids waiting on their own clusters must not share the device at once (each
    // could hold SMs the other needs): within the process they run one at a time per device.
    static std::mutex coop_mu[64];
    std::lock_guard<std::mutex> guard(coop_mu[current_device() & 63]);
    cudaError_t e = cudaMemsetAsync(M.glm_cnt, 0, sizeof(unsigned int) * tiles * 16, st);
    if (e != cudaSuccess) return e;
    e = launch(0, tiles, cs, nc);
    if (verbose)
      std::fprintf(stderr, "glm_kernel<%d,%d>: %d tiles x %d clusters of %d CTAs: %s\n", FAM, KP, tiles, nc, cs,
                   cudaGetErrorString(e));
    if (e == cudaSuccess) return cudaStreamSynchronize(st);  // a kernel fault is returned, not retried
    cudaGetLastError();  // not co-residentable as one cooperative grid: one cluster per tile
    --sampler_launch_count();
    nc = 1;
    cs = cs_single;
  }
  if (verbose)
    std::fprintf(stderr, "glm_kernel<%d,%d>: %d tiles, cluster %d (active clusters: 8 -> %d, 16 -> %d)\n", FAM, KP,
                 tiles, cs, fits(8), fits(16));
  const int sms = glm_sm_count();
  static const bool no_split = std::getenv("PCVG_NO_TAIL_SPLIT") != nullptr;  // A/B tests only
  if (cs == 1 && tiles > sms && tiles % sms != 0 && !no_split) {
    // Wave tail: one CTA per SM per wave, so the last partial wave of r tiles would take as long
    // as a full one. Its tiles run instead as row-split clusters of up to 8 CTAs (the cluster
    // path of the few-chain configurations). Their X^T R sums are split by rank and combined in a
    // different order than the unsplit quarter sums, so tail chains agree with an unsplit launch to
    // rounding only (test_wave_tail_split_matches_unsplit); full-wave chains are bit-identical.
    const int r = tiles % sms, ntiles_rows = (M.n + Geom<KP>::TM - 1) / Geom<KP>::TM;
    int ct = 1;
    // double the cluster while the tail still fits on the SMs in one round: all r clusters must be
    // co-resident (a cluster fits within one GPC), else the last ones wait for a second round
    while (ct < 8 && r * ct * 2 <= sms && ntiles_rows >= 4 * ct * 2 && fits(ct * 2) >= r) ct *= 2;
    cudaError_t e = launch(0, tiles - r, 1, 1);
    if (e != cudaSuccess) return e;
    return launch(tiles - r, r, ct, 1);
  }
  return launch(0, tiles, cs, 1);
}


}  // namespace

int glm_sm_count() { return device_sm_count(); }

// Cluster size: enough CTAs per 64-chain tile to cover the GPU, at most 16 (non-portable; the
// launcher caps it at 8 where the device cannot schedule 16), and at least two row tiles per CTA.
int glm_cluster_size(int n, int kp, int nch) {
  const int tm = kp <= 8 ? 256 : (kp <= 16 ? 128 : 64);
  const int tiles = (nch + kC - 1) / kC;
  const int ntiles = (n + tm - 1) / tm;
  const int sms = device_sm_count();
  int cs = 1;
  while (cs < 16 && tiles * cs * 2 <= sms && ntiles >= 4 * cs) cs *= 2;
  // 16-CTA clusters only for the fewest tiles (cfg2 K-fold: 2, Step 1: 1): at most 7 fit at once,
  // and two models' launches run concurrently (cfg4 under ROWS: 7 tiles stays at 8, 0.85M vs 0.61M)
  if (cs == 16 && tiles * 16 > 64) cs = 8;
  return cs;
}

// Clusters per chain tile for the few-chain launches: when 16-CTA clusters still leave most SMs
// idle (cfg2 K-fold: two tiles on 32 of 148 SMs; Step 1: one tile), each tile is split over nc
// clusters whose sums meet in global memory (reduce_clusters), keeping >= 2 row tiles per CTA.
int glm_clusters_per_tile(int n, int kp, int nch, int cs, bool have_scratch) {
  static const bool off = std::getenv("PCVG_NO_MULTICLUSTER") != nullptr;  // A/B tests only
  if (off || !have_scratch || cs < 8) return 1;
  const int tm = kp <= 8 ? 256 : (kp <= 16 ? 128 : 64);
  const int tiles = (nch + kC - 1) / kC;
  const int ntiles = (n + tm - 1) / tm;
  // up to kMaxClusters per tile, at least one row tile per CTA (a single tile - Step 1 - splits its
  // 157 row tiles over up to 120 CTAs: 2 per CTA instead of 3 at 8 clusters)
  int nc = std::min(kMaxClusters, device_sm_count() / (tiles * cs));
  while (nc > 1 && ntiles < cs * nc) --nc;
  return std::max(nc, 1);
}

// Scratch of the multi-cluster launches of a model with nch chains: partial doubles and counters.
void glm_multicluster_scratch(int kp, int nch, size_t* part_doubles, size_t* counters) {
  const int tiles = (nch + kC - 1) / kC;
  *part_doubles = static_cast<size_t>(tiles) * 2 * kMaxClusters * (static_cast<size_t>(kp) * kC + kC);
  *counters = static_cast<size_t>(tiles) * 16;  // one per (tile, cluster rank)
}

// Padded design width for a model on the tensor-core path, or 0 if it does not qualify
// (hierarchical families with J > 1 use gauss_kernel).
int glm_width(int family, int J, int nc) {
  const int cols = nc + 1;  // intercept + covariates
  if (family == kLogistic) return cols <= 8 ? 8 : (cols <= 16 ? 16 : (cols <= 52 ? 52 : 0));
  if (family == kGrouped && J == 1) return cols <= 8 ? 8 : (cols <= 16 ? 16 : 0);
  if (family == kSeasonal) return cols <= 8 ? 8 : (cols <= 16 ? 16 : 0);
  return 0;
}

cudaError_t launch_glm(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st) {
  switch (M.family * 100 + M.nc_pad) {
    case kLogistic * 100 + 8: return launch_t<kLogistic, 8>(M, S, A, st);
    case kLogistic * 100 + 16: return launch_t<kLogistic, 16>(M, S, A, st);
    case kLogistic * 100 + 52: return launch_t<kLogistic, 52>(M, S, A, st);
    case kGrouped * 100 + 8: return launch_t<kGrouped, 8>(M, S, A, st);
    case kGrouped * 100 + 16: return launch_t<kGrouped, 16>(M, S, A, st);
    case kSeasonal * 100 + 8: return launch_t<kSeasonal, 8>(M, S, A, st);
    case kSeasonal * 100 + 16: return launch_t<kSeasonal, 16>(M, S, A, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pcvg
