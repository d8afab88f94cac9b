// Fused HMC kernel for the Gaussian linear families (sm_100a, FP64):
//   grouped regression  (grouped_regression.cpp:56-163)  - cfg1 (J=1), paper Ex-1
//   radon-style         (radon.cpp:50-138)                - cfg3
//   seasonal AR         (seasonal_ar.cpp:37-115)          - cfg4 (time-block / hv-block folds)
//
// All three share one per-observation form: m_i = off(g_i) + sum_c w_c x_ic, r_i = y_i - m_i,
// and a gradient built from the masked sums S_r[g], S_xr[c], S_rr. One chain is owned by T
// consecutive lanes (T | 32); the lanes split the observations of every group segment and
// butterfly-reduce the sums, so each lane ends with identical gradient bits and advances an
// identical copy of the chain's global parameters (kept in registers). Group parameters live in
// HBM as [dim][chain] arrays (coalesced across the chains of a warp) and are updated group by
// group inside the gradient pass. Per HMC transition (hmc.cpp:53-99) the kernel runs n_lf
// gradient passes (the gradient and log joint at the current position are cached - the reference
// recomputes the identical bits, hmc.cpp:37,69-70 - and the proposal's log joint is fused into
// the last pass), the Metropolis test, log_pred and the online accumulator update
// (accum.cpp:164-182). Chains are independent; a CTA holds 128/T chains.
#pragma once
#include <math_constants.h>

#include <cstdlib>

#include "device_cache.hpp"
#include "device_common.cuh"
#include "score_extra.cuh"
#include "tc_common.cuh"
#include "types.cuh"

namespace pcvg {

namespace {

constexpr int kBlock = 128;

template <int T>
__device__ __forceinline__ double lane_sum(double v, unsigned mask) {
#pragma unroll
  for (int off = T / 2; off > 0; off >>= 1) v += __shfl_xor_sync(mask, v, off, T);
  return v;
}

__device__ __forceinline__ double logistic_fn(double u) { return 1.0 / (1.0 + exp(-u)); }

// Normals of one HMC momentum refresh read from a snapshot of the chain stream by dimension
// index: normal i of this transition, honouring a Box-Muller variate cached by the previous
// transition (rng.hpp:75-87). Lets the group momenta be generated inside the first gradient pass.
struct NormalCursor {
  uint64_t pos0;
  bool hc0;
  double c0;
  int64_t pair;
  double ncos, nsin;

  __device__ void start(const ChainRng& R) {
    pos0 = R.pos;
    hc0 = R.has_cached;
    c0 = R.cached;
    pair = -1;
  }
  __device__ double at(ChainRng& R, int i) {
    if (hc0) {
      if (i == 0) return c0;
      i -= 1;
    }
    const int64_t pr = i >> 1;
    if (pr != pair) {  // the pair R.normal() would draw at this stream position (same bits)
      normal_pair_at(R.k0, R.k1, R.stream, pos0 + 4 * static_cast<uint64_t>(pr), &ncos, &nsin);
      pair = pr;
    }
    return (i & 1) ? nsin : ncos;
  }
  // Leaves R exactly where the reference stream is after d normal() calls.
  __device__ void finish(ChainRng& R, int d) {
    if (d == 0) return;
    const int m = hc0 ? d - 1 : d;  // normals drawn from fresh pairs
    const int64_t pairs = (m + 1) / 2;
    if (m & 1) {
      R.cached = at(R, d);  // the sin half of the last pair
      R.has_cached = true;
    } else {
      R.has_cached = false;
    }
    R.pos = pos0 + 4 * static_cast<uint64_t>(pairs);
  }
};

// Per-pass quantities derived from the global parameters.
template <int NCM>
struct Prep {
  double w[NCM];  // covariate weights
  double off0;    // offset without the group term
  double v, inv_v, logv;
  double va, sa;  // group scale (grouped: va = sig_a^2; radon: va, sa = sqrt(va))
  double inv_va;  // 1 / va (the sufficient-statistics passes multiply instead of dividing)
  double vb;      // rat M_A: slope scale s_b^2
};

// Register slot -> global parameter index. Slots put the parameters whose position depends
// on runtime sizes (P, p, q) at fixed registers so no register array is indexed dynamically:
//   grouped  [mu_alpha, log sigma_alpha, log sigma_y, beta_0..beta_{P-1}]
//   radon    [beta, mu_alpha, log sigma_alpha^2, log sigma_y^2]           (reference order)
//   rat M_B  [beta, mu_a, log s_a, log s_y]; rat M_A [mu_a, mu_b, log s_a, log s_b, log s_y]
//   seasonal [beta_0, log sigma, cov 0..p+q-1 -> u_1..u_p, beta_1..beta_q]
template <int FAM>
__device__ __forceinline__ int gidx(const ModelDev& M, int r) {
  if constexpr (FAM == kGrouped) return r < 3 ? M.nc + r : r - 3;
  else if constexpr (FAM == kRadon || FAM == kRatA || FAM == kRatB) return r;
  else return r == 0 ? M.p : (r == 1 ? M.p + M.q + 1 : (r - 2 < M.p ? r - 2 : r - 1));
}

template <int FAM, int NCM, int NGM>
__device__ __forceinline__ void prepare(const ModelDev& M, const double* qG, Prep<NCM>& P) {
  if constexpr (FAM == kGrouped) {
#pragma unroll
    for (int c = 0; c < NCM; ++c) P.w[c] = (c < M.nc) ? M.cmask[c] * qG[3 + c] : 0.0;
    const double sig_a = exp(qG[1]);
    const double sig_y = exp(qG[2]);
    P.va = sig_a * sig_a;
    P.v = sig_y * sig_y;
    P.off0 = 0.0;
  } else if constexpr (FAM == kRadon) {
    P.w[0] = M.include_floor ? qG[0] : 0.0;
    P.off0 = qG[1];
    P.va = exp(qG[2]);
    P.sa = sqrt(P.va);
    P.v = exp(qG[3]);
  } else if constexpr (FAM == kRatB) {  // rat_growth.cpp:148-172
    P.w[0] = qG[0];
    P.off0 = 0.0;
    const double s_a = exp(qG[2]), s_y = exp(qG[3]);
    P.va = s_a * s_a;
    P.v = s_y * s_y;
  } else if constexpr (FAM == kRatA) {  // rat_growth.cpp:117-147 (slope per group)
    P.w[0] = 0.0;
    P.off0 = 0.0;
    const double s_a = exp(qG[2]), s_b = exp(qG[3]), s_y = exp(qG[4]);
    P.va = s_a * s_a;
    P.vb = s_b * s_b;
    P.v = s_y * s_y;
  } else {  // seasonal
#pragma unroll
    for (int c = 0; c < NCM; ++c) {
      if (c < M.p) {
        const double w = logistic_fn(qG[2 + c]);
        P.w[c] = M.rho_sym ? 2.0 * w - 1.0 : 0.5 * (1.0 + w);
      } else {
        P.w[c] = c < M.p + M.q ? qG[2 + c] : 0.0;
      }
    }
    P.off0 = qG[0];
    const double sigma = exp(qG[1]);
    P.v = sigma * sigma;
  }
  P.inv_v = 1.0 / P.v;
  if constexpr (FAM != kSeasonal) P.inv_va = 1.0 / P.va;  // used by the RCP passes only (else eliminated)
  P.logv = log(P.v);
}

template <int FAM, int NCM>
__device__ __forceinline__ double group_offset(const Prep<NCM>& P, double qg) {
  if constexpr (FAM == kGrouped || FAM == kRatA || FAM == kRatB) return qg;
  else if constexpr (FAM == kRadon) return P.off0 + P.sa * qg;
  else return P.off0;
}

// Replicated (not lane-reduced) per-group accumulators.
struct GroupAcc {
  double a0, a1, a2, a3;
};

// a / v, or a * (1 / v) in the sufficient-statistics passes (RCP: one rounding more, no division)
template <bool RCP>
__device__ __forceinline__ double dv(double a, double v, double inv) {
  if constexpr (RCP) return a * inv;
  else return a / v;
}

// d log p / d q_g given the lane-reduced residual sum of group g; updates replicated sums.
template <int FAM, int NCM, int NGM, bool RCP = false>
__device__ __forceinline__ double group_grad(const Prep<NCM>& P, const double* qG,
                                            const ModelDev& M, double qg, double srg,
                                            GroupAcc& G) {
  if constexpr (FAM == kGrouped) {  // grouped_regression.cpp:100-116
    const double dev = qg - qG[0];
    G.a0 += dv<RCP>(dev, P.va, P.inv_va);  // -> d/d mu_alpha
    G.a1 += dev * dev;   // -> d/d log sigma_alpha, prior
    return dv<RCP>(srg, P.v, P.inv_v) - dv<RCP>(dev, P.va, P.inv_va);
  } else if constexpr (FAM == kRatB || FAM == kRatA) {  // rat_growth.cpp:129-137, 159-164 (alpha_g)
    const double dev = qg - (FAM == kRatB ? qG[1] : qG[0]);
    G.a0 += dv<RCP>(dev, P.va, P.inv_va);  // -> d/d mu_a
    G.a1 += dev * dev;   // -> d/d log s_a, prior
    return dv<RCP>(srg, P.v, P.inv_v) - dv<RCP>(dev, P.va, P.inv_va);
  } else {  // radon.cpp:93-105
    G.a0 += srg;       // sum r (-> d/d mu_alpha)
    G.a1 += srg * qg;  // sum r z (-> d/d log va)
    G.a2 += qg * qg;   // prior on z
    return dv<RCP>(P.sa * srg, P.v, P.inv_v) - qg;
  }
}

// Global gradient and (optionally) log joint from the reduced sums.
template <int FAM, int NCM, int NGM, bool RCP = false>
__device__ __forceinline__ void global_grad(const ModelDev& M, const Prep<NCM>& P,
                                            const double* qG, const double* sxr, double sr,
                                            double srr, const GroupAcc& G, int n_train,
                                            double* gG, bool value, double& lp) {
  const double ntr = static_cast<double>(n_train);
  if constexpr (FAM == kGrouped) {  // grouped_regression.cpp:109-121, 65-85
#pragma unroll
    for (int c = 0; c < NCM; ++c)
      if (c < M.nc) gG[3 + c] = M.cmask[c] * dv<RCP>(sxr[c], P.v, P.inv_v) - qG[3 + c];
    gG[0] = G.a0 - qG[0];
    gG[1] = dv<RCP>(G.a1, P.va, P.inv_va) - M.J - P.va * 0.1 + 1.0;  // half-normal(0, 10) prior: v / 10
    gG[2] = dv<RCP>(srr, P.v, P.inv_v) - ntr - P.v * 0.1 + 1.0;
    if (value) {
      double l = -0.5 * (ntr * (kLog2Pi + P.logv) + srr / P.v);
      l += -0.5 * (M.J * (kLog2Pi + log(P.va)) + G.a1 / P.va);
      l += -0.5 * (kLog2Pi + qG[0] * qG[0]);
#pragma unroll
      for (int c = 0; c < NCM; ++c)
        if (c < M.nc) l += -0.5 * (kLog2Pi + qG[3 + c] * qG[3 + c]);
      const double sig_a = exp(qG[1]), sig_y = exp(qG[2]);
      l += M.c_lhn10 - sig_a * sig_a / 20.0 + qG[1];
      l += M.c_lhn10 - sig_y * sig_y / 20.0 + qG[2];
      lp = l;
    }
  } else if constexpr (FAM == kRadon) {  // radon.cpp:102-106, 50-74
    gG[0] = (M.include_floor ? dv<RCP>(sxr[0], P.v, P.inv_v) : 0.0) - qG[0];
    gG[1] = dv<RCP>(G.a0, P.v, P.inv_v) - qG[1] / 4.0;
    gG[2] = dv<RCP>(0.5 * P.sa * G.a1, P.v, P.inv_v) + 6.0 - 9.0 * P.va;
    gG[3] = 0.5 * (dv<RCP>(srr, P.v, P.inv_v) - ntr) + 10.0 - 10.0 * P.v;
    if (value) {
      double l = -0.5 * (ntr * (kLog2Pi + P.logv) + srr / P.v);
      l += -0.5 * (M.J * kLog2Pi + G.a2);
      l += -0.5 * (kLog2Pi + qG[0] * qG[0]);
      l += -0.5 * (kLog2Pi + M.c_log4 + qG[1] * qG[1] / 4.0);
      l += M.c_lgamma6_9 + 5.0 * qG[2] - 9.0 * P.va + qG[2];
      l += M.c_lgamma10_10 + 9.0 * qG[3] - 10.0 * P.v + qG[3];
      lp = l;
    }
  } else if constexpr (FAM == kRatB) {  // rat_growth.cpp:148-172, 88-107
    const double s_a = exp(qG[2]), s_y = exp(qG[3]);
    gG[0] = dv<RCP>(sxr[0], P.v, P.inv_v) - (qG[0] - 6.0) / 2.0;
    gG[1] = G.a0 - (qG[1] - 250.0) / 20.0;
    gG[2] = dv<RCP>(G.a1, P.va, P.inv_va) - M.J + 25.0 - 2.0 * s_a;
    gG[3] = dv<RCP>(srr, P.v, P.inv_v) - ntr + 1.0 - 2.0 * s_y;
    if (value) {
      double l = -0.5 * (ntr * (kLog2Pi + P.logv) + srr / P.v);
      l += -0.5 * (M.J * (kLog2Pi + log(P.va)) + G.a1 / P.va);
      const double d6 = qG[0] - 6.0, d250 = qG[1] - 250.0;
      l += -0.5 * (kLog2Pi + M.c_log2 + d6 * d6 / 2.0);
      l += -0.5 * (kLog2Pi + M.c_log20 + d250 * d250 / 20.0);
      l += M.c_lg25_2 + 25.0 * qG[2] - 2.0 * s_a;
      l += M.c_lg1_2 + 1.0 * qG[3] - 2.0 * s_y;
      lp = l;
    }
  } else if constexpr (FAM == kRatA) {  // rat_growth.cpp:117-147, 72-87
    const double s_a = exp(qG[2]), s_b = exp(qG[3]), s_y = exp(qG[4]);
    gG[0] = G.a0 - (qG[0] - 250.0) / 20.0;
    gG[1] = G.a2 - (qG[1] - 6.0) / 2.0;
    gG[2] = G.a1 / P.va - M.J + 25.0 - 2.0 * s_a;
    gG[3] = G.a3 / P.vb - M.J + 5.0 - 10.0 * s_b;
    gG[4] = srr / P.v - ntr + 1.0 - 2.0 * s_y;
    if (value) {
      double l = -0.5 * (ntr * (kLog2Pi + P.logv) + srr / P.v);
      l += -0.5 * (M.J * (kLog2Pi + log(P.va)) + G.a1 / P.va);
      l += -0.5 * (M.J * (kLog2Pi + log(P.vb)) + G.a3 / P.vb);
      const double d250 = qG[0] - 250.0, d6 = qG[1] - 6.0;
      l += -0.5 * (kLog2Pi + M.c_log20 + d250 * d250 / 20.0);
      l += -0.5 * (kLog2Pi + M.c_log2 + d6 * d6 / 2.0);
      l += M.c_lg25_2 + 25.0 * qG[2] - 2.0 * s_a;
      l += M.c_lg5_10 + 5.0 * qG[3] - 10.0 * s_b;
      l += M.c_lg1_2 + 1.0 * qG[4] - 2.0 * s_y;
      lp = l;
    }
  } else {  // seasonal_ar.cpp:79-105, 59-77
    double l = 0.0;
#pragma unroll
    for (int c = 0; c < NCM; ++c) {
      if (c < M.p) {
        const double w = logistic_fn(qG[2 + c]);
        const double dw = w * (1.0 - w);
        const double drho = M.rho_sym ? 2.0 * dw : 0.5 * dw;
        gG[2 + c] = dv<RCP>(sxr[c] * drho, P.v, P.inv_v) + (4.0 * (1.0 - w) - 4.0 * w + 1.0 - 2.0 * w);
        if (value) l += 4.0 * log(w) + 4.0 * log1p(-w) + M.c_lbeta55 + log(w) + log1p(-w);
      } else if (c < M.p + M.q) {
        gG[2 + c] = dv<RCP>(sxr[c], P.v, P.inv_v) - qG[2 + c];
        if (value) l += -0.5 * (kLog2Pi + qG[2 + c] * qG[2 + c]);
      }
    }
    gG[0] = dv<RCP>(sr, P.v, P.inv_v) - qG[0];
    gG[1] = dv<RCP>(srr, P.v, P.inv_v) - ntr - P.v + 1.0;
    if (value) {
      l += -0.5 * (ntr * (kLog2Pi + P.logv) + srr / P.v);
      l += -0.5 * (kLog2Pi + qG[0] * qG[0]);
      const double sigma = exp(qG[1]);
      l += M.c_lhn1 - sigma * sigma / 2.0 + qG[1];
      lp = l;
    }
  }
}

// One gradient evaluation at (qG, group params) for chain c. kind: 0 = evaluate at the stored
// position (no dynamics), 1 = first leapfrog step (fuses momentum draw + half kick + drift of
// the group dims), 2 = later steps. On leapfrog kinds the group momenta get the kick `scale`.
template <int FAM, int T, int NCM, int NGM, bool VALUE>
__device__ __forceinline__ void grad_pass(const ModelDev& M, const ChainsDev& S, int c, int t,
                                          unsigned mask, int lo, int hi, int n_train,
                                          const double* qG, int kind, bool last, double scale,
                                          int cur, NormalCursor& nc, ChainRng& R,
                                          const double* probe_p, double* gG, double& lp,
                                          double& k0g, double& k1g, bool& bad) {
  Prep<NCM> P;
  prepare<FAM, NCM, NGM>(M, qG, P);
  const int n = M.n;
  const int nch = S.nch;
  const double eps = M.step, half = 0.5 * M.step;
  const size_t plane = static_cast<size_t>(M.dim) * nch;
  double sxr[NCM];
#pragma unroll
  for (int k = 0; k < NCM; ++k) sxr[k] = 0.0;
  double sr_tot = 0.0, srr = 0.0;
  bool poison = false;
  GroupAcc G{0.0, 0.0, 0.0, 0.0};
  const int ngroups = M.J > 0 ? M.J : 1;
  for (int g = 0; g < ngroups; ++g) {
    double qg = 0.0, pg = 0.0;
    const int r0 = M.J > 0 ? __ldg(M.grp_ptr + g) : 0;
    const int r1 = M.J > 0 ? __ldg(M.grp_ptr + g + 1) : n;
    const size_t gi = static_cast<size_t>(g) * nch + c;
    if constexpr (FAM != kSeasonal) {
      const double mg = __ldg(M.inv_mass + g);
      if (kind == 0) {
        qg = S.pos[cur * plane + gi];
      } else if (kind == 1) {
        const double p0 = probe_p ? probe_p[static_cast<size_t>(c) * M.dim + g]
                                  : nc.at(R, g) / sqrt(mg);
        k0g += mg * p0 * p0;
        pg = p0 + half * S.grad[cur * plane + gi];
        qg = S.pos[cur * plane + gi] + eps * mg * pg;
      } else {
        pg = S.wp[gi];
        qg = S.pos[(cur ^ 1) * plane + gi] + eps * mg * pg;
      }
      bad |= !isfinite(qg);
    }
    const double off = group_offset<FAM, NCM>(P, qg);
    double srg = 0.0;
    for (int i = r0 + t; i < r1; i += T) {
      const double yi = __ldg(M.y + i);
      const int ki = __ldg(M.key + i);
      double m = off;
      double xs[NCM];
#pragma unroll
      for (int k = 0; k < NCM; ++k) {
        if (k < M.nc) {
          xs[k] = __ldg(M.x + static_cast<size_t>(k) * n + i);
          m = fma(P.w[k], xs[k], m);
        } else {
          xs[k] = 0.0;
        }
      }
      const double r = yi - m;
      const bool train = static_cast<unsigned>(ki - lo) >= static_cast<unsigned>(hi - lo);
      const double wr = train ? r : 0.0;
      srg += wr;
#pragma unroll
      for (int k = 0; k < NCM; ++k) sxr[k] = fma(xs[k], wr, sxr[k]);
      srr = fma(wr, r, srr);
      if (VALUE && !train) poison |= !isfinite(P.logv + r * r * P.inv_v);
    }
    if constexpr (FAM != kSeasonal) {
      srg = lane_sum<T>(srg, mask);
      const double gg = group_grad<FAM, NCM, NGM>(P, qG, M, qg, srg, G);
      if (kind == 0) {
        if (t == 0) S.grad[cur * plane + gi] = gg;
        bad |= !isfinite(gg);
      } else {
        bad |= !isfinite(gg);
        pg += scale * gg;
        bad |= !isfinite(pg);
        if (t == 0) {
          S.pos[(cur ^ 1) * plane + gi] = qg;
          S.wp[gi] = pg;
          if (last) S.grad[(cur ^ 1) * plane + gi] = gg;
        }
        if (last) k1g += __ldg(M.inv_mass + g) * pg * pg;
      }
    } else {
      sr_tot += srg;
    }
  }
#pragma unroll
  for (int k = 0; k < NCM; ++k) sxr[k] = lane_sum<T>(sxr[k], mask);
  srr = lane_sum<T>(srr, mask);
  if constexpr (FAM == kSeasonal) sr_tot = lane_sum<T>(sr_tot, mask);
  if (VALUE) {
    // any lane's poisoned test row poisons the chain (0 * non-finite = NaN, grouped_regression.cpp:74-76)
    const unsigned any = __ballot_sync(mask, poison);
    poison = any != 0;
  }
  global_grad<FAM, NCM, NGM>(M, P, qG, sxr, sr_tot, srr, G, n_train, gG, VALUE, lp);
  if (VALUE && poison) lp = CUDART_NAN;
  __syncwarp(mask);  // group-dim stores of lane 0 become visible to the chain's lanes
}

// Position + momentum slot arrays per group parameter kind (rat M_A: intercepts and slopes).
__host__ __device__ inline int suff_slot_arrays(const ModelDev& M) { return M.family == kRatA ? 4 : 2; }

// Shared-memory group slots of the sufficient-statistics kernel (position + momentum per owned
// group, [slot][kBlock] doubles each): warp-per-chain launches of hierarchical models whose slots
// fit; 0 = the group state goes through the HBM planes.
__host__ __device__ inline int suff_slots(const ModelDev& M, int T) {
  if (T != 32 || M.J < 2) return 0;
  const int ns = (M.J + 31) / 32;
  return suff_slot_arrays(M) * ns * kBlock * 8 <= 96 * 1024 ? ns : 0;
}

// grad_pass on the fold's sufficient statistics (suffstats.cpp; NB < 0): the same masked sums
// S_r[g], S_xr, S_rr as the row loop, from the packed training Gram A_k and the group sums s_g, in
// O(d^2 + J d) instead of O(n d) per pass. u = (y, x), om = (1, -w):
//   S_r[g] = om.s_g - n_g off_g;  S_xr = (A om)[1..] - sum_g off_g s_g[1..];
//   S_rr = om^T A om - sum_g off_g (om.s_g + S_r[g]).
// T lanes per chain split the Gram entries and the groups (lane t owns groups t, t + T, ...) and
// butterfly-reduce the partial sums, so every lane ends with identical bits. With `qs` (T = 32,
// hierarchical), a lane keeps its groups' position / momentum in shared-memory slots across the
// passes of a transition (slot j of group t + 32 j at qs[j * kBlock]); the planes are written in
// the last pass only. The value pass also evaluates the fold's excluded rows for the reference's
// poisoning of a non-finite masked term (grouped_regression.cpp:74-76).
// Rat growth M_A (per-subject slope beta_g, rat_growth.cpp:117-147): every sum is per subject,
// from the subject's (y, t) Gram (sgA / sov_A) and sums: om_g = (1, -beta_g),
//   S_r[g] = om_g.s_g - n_g alpha_g, S_tr[g] = (A_g om_g)[1] - alpha_g s_g[1],
//   S_rr = sum_g om_g^T A_g om_g - alpha_g (om_g.s_g + S_r[g]).
template <int FAM, int T, int NCM, int NGM, bool VALUE>
__device__ __forceinline__ void suff_pass(const ModelDev& M, const ChainsDev& S, int c, int t, unsigned mask,
                                          int fold, int n_train, const double* qG, int kind, bool last,
                                          double scale, int cur, NormalCursor& nc, ChainRng& R,
                                          const double* probe_p, double* gG, double& lp, double& k0g,
                                          double& k1g, bool& bad, double* qs, double* ps) {
  constexpr int D = NCM + 1;
  Prep<NCM> P;
  prepare<FAM, NCM, NGM>(M, qG, P);
  const int nch = S.nch;
  const int d = M.nc + 1;
  const double eps = M.step, half = 0.5 * M.step;
  const size_t plane = static_cast<size_t>(M.dim) * nch;
  // om[i] = 1 (i = 0), -w[i - 1] (w = 0 past nc)
#define PCVG_OM(i) ((i) == 0 ? 1.0 : -P.w[(i) - 1])
  // this lane's share of q = A om over the packed lower triangle (row i at i (i + 1) / 2)
  const double* A = M.sA + static_cast<size_t>(fold) * M.sdp;
  double q[D];
#pragma unroll
  for (int i = 0; i < D; ++i) q[i] = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    if (FAM != kRatA && i < d) {
#pragma unroll
      for (int j = 0; j <= i; ++j) {
        const int e = i * (i + 1) / 2 + j;
        if (T == 1 || e % T == t) {
          const double a = __ldg(A + e);
          q[i] = fma(a, PCVG_OM(j), q[i]);
          if (j < i) q[j] = fma(a, PCVG_OM(i), q[j]);
        }
      }
    }
  }
  double sv[D];  // this lane's sum_g off_g s_g
#pragma unroll
  for (int i = 0; i < D; ++i) sv[i] = 0.0;
  // centred statistics (suffstats.cpp): offsets shift by om.ubar, S_xr gains ubar_x * sum_g S_r[g]
  double om_u = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i)
    if (i < d) om_u = fma(PCVG_OM(i), M.su[i], om_u);
  double t2 = 0.0, sr_tot = 0.0, sr_all = 0.0, dk0 = 0.0, dk1 = 0.0, srr_a = 0.0;
  GroupAcc G{0.0, 0.0, 0.0, 0.0};
  // rat M_A: slope slots after the intercept slots
  const int ns_a = FAM == kRatA && qs ? suff_slots(M, T) : 0;
  double* qs2 = qs ? qs + 2 * static_cast<size_t>(ns_a) * kBlock : nullptr;
  double* ps2 = qs ? qs + 3 * static_cast<size_t>(ns_a) * kBlock : nullptr;
  const int ov0 = __ldg(M.sov_ptr + fold), ov_end = __ldg(M.sov_ptr + fold + 1);
  int ov = ov0;
  // the group of the next override entry, held in a register: the walk loads sov_g only when it
  // advances (once per override), not twice per group (cfg3: 14% of the stall samples)
  int ovg = ov < ov_end ? __ldg(M.sov_g + ov) : 0x7fffffff;
  const int ngroups = M.J > 0 ? M.J : 1;
  for (int g = t, jj = 0; g < ngroups; g += T, ++jj) {
    double qg = 0.0, pg = 0.0;
    const size_t gi = static_cast<size_t>(g) * nch + c;
    if constexpr (FAM != kSeasonal) {
      const double mg = __ldg(M.inv_mass + g);
      if (kind == 0) {
        qg = S.pos[cur * plane + gi];
      } else if (kind == 1) {
        const double p0 = probe_p ? probe_p[static_cast<size_t>(c) * M.dim + g] : nc.at(R, g) / sqrt(mg);
        dk0 += mg * p0 * p0;
        pg = p0 + half * S.grad[cur * plane + gi];
        qg = S.pos[cur * plane + gi] + eps * mg * pg;
      } else if (qs) {
        pg = ps[jj * kBlock];
        qg = qs[jj * kBlock] + eps * mg * pg;
      } else {
        pg = S.wp[gi];
        qg = S.pos[(cur ^ 1) * plane + gi] + eps * mg * pg;
      }
      bad |= !isfinite(qg);
    }
    const double off = group_offset<FAM, NCM>(P, qg) - om_u;
    // this fold's statistics of group g: an override when the fold holds out some of its rows
    while (ovg < g) {
      ++ov;
      ovg = ov < ov_end ? __ldg(M.sov_g + ov) : 0x7fffffff;
    }
    double ng;
    const double* sp;
    const double* Ag = nullptr;  // rat M_A: the subject's (y, t) Gram
    if (ovg == g) {
      ng = __ldg(M.sov_n + ov);
      sp = M.sov_s + static_cast<size_t>(ov) * d;
      if constexpr (FAM == kRatA) Ag = M.sov_A + static_cast<size_t>(ov) * 3;
    } else {
      ng = __ldg(M.sgn + g);
      sp = M.sgs + static_cast<size_t>(g) * d;
      if constexpr (FAM == kRatA) Ag = M.sgA + static_cast<size_t>(g) * 3;
    }
    if constexpr (FAM == kRatA) {  // per-subject slope beta_g (dim J + g), its own slots
      const int gs = M.J + g;
      const size_t si = static_cast<size_t>(gs) * nch + c;
      const double ms = __ldg(M.inv_mass + gs);
      double qb = 0.0, pb = 0.0;
      if (kind == 0) {
        qb = S.pos[cur * plane + si];
      } else if (kind == 1) {
        const double p0 = probe_p ? probe_p[static_cast<size_t>(c) * M.dim + gs] : nc.at(R, gs) / sqrt(ms);
        dk0 += ms * p0 * p0;
        pb = p0 + half * S.grad[cur * plane + si];
        qb = S.pos[cur * plane + si] + eps * ms * pb;
      } else if (qs) {
        pb = ps2[jj * kBlock];
        qb = qs2[jj * kBlock] + eps * ms * pb;
      } else {
        pb = S.wp[si];
        qb = S.pos[(cur ^ 1) * plane + si] + eps * ms * pb;
      }
      bad |= !isfinite(qb);
      const double sy = __ldg(sp), st = __ldg(sp + 1);
      const double ayy = __ldg(Ag), aty = __ldg(Ag + 1), att = __ldg(Ag + 2);
      const double ws = fma(-qb, st, sy);
      const double srg = fma(-ng, qg, ws);
      const double str = fma(-qb, att, aty) - qg * st;  // sum t r
      srr_a += (ayy - 2.0 * qb * aty + qb * qb * att) - qg * (ws + srg);
      const double db = qb - qG[1];  // beta_g - mu_b
      G.a2 += db / P.vb;
      G.a3 += db * db;
      const double gsl = dv<true>(str, P.v, P.inv_v) - db / P.vb;  // rat_growth.cpp:127-137
      bad |= !isfinite(gsl);
      if (kind == 0) {
        S.grad[cur * plane + si] = gsl;
      } else {
        pb += scale * gsl;
        bad |= !isfinite(pb);
        if (qs && !last) {
          qs2[jj * kBlock] = qb;
          ps2[jj * kBlock] = pb;
        } else {
          S.pos[(cur ^ 1) * plane + si] = qb;
          S.wp[si] = pb;
        }
        if (last) {
          S.grad[(cur ^ 1) * plane + si] = gsl;
          dk1 += ms * pb * pb;
        }
      }
      const double gg = group_grad<FAM, NCM, NGM, true>(P, qG, M, qg, srg, G);  // alpha_g
      bad |= !isfinite(gg);
      if (kind == 0) {
        S.grad[cur * plane + gi] = gg;
      } else {
        pg += scale * gg;
        bad |= !isfinite(pg);
        if (qs && !last) {
          qs[jj * kBlock] = qg;
          ps[jj * kBlock] = pg;
        } else {
          S.pos[(cur ^ 1) * plane + gi] = qg;
          S.wp[gi] = pg;
        }
        if (last) {
          S.grad[(cur ^ 1) * plane + gi] = gg;
          dk1 += __ldg(M.inv_mass + g) * pg * pg;
        }
      }
      continue;
    }
    double ws = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      if (i < d) {
        const double si = __ldg(sp + i);
        ws = fma(PCVG_OM(i), si, ws);
        if (i > 0) sv[i] = fma(off, si, sv[i]);
      }
    }
    const double srg = fma(-ng, off, ws);
    t2 = fma(off, ws + srg, t2);
    sr_all += srg;
    if constexpr (FAM != kSeasonal) {
      const double gg = group_grad<FAM, NCM, NGM, true>(P, qG, M, qg, srg, G);
      bad |= !isfinite(gg);
      if (kind == 0) {
        S.grad[cur * plane + gi] = gg;
      } else {
        pg += scale * gg;
        bad |= !isfinite(pg);
        if (qs && !last) {
          qs[jj * kBlock] = qg;
          ps[jj * kBlock] = pg;
        } else {
          S.pos[(cur ^ 1) * plane + gi] = qg;
          S.wp[gi] = pg;
        }
        if (last) {
          S.grad[(cur ^ 1) * plane + gi] = gg;
          dk1 += __ldg(M.inv_mass + g) * pg * pg;
        }
      }
    } else {
      sr_tot += srg;
    }
  }
  // lane partials -> identical totals on every lane (xor butterfly)
  double quad = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) quad = fma(PCVG_OM(i), q[i], quad);
#undef PCVG_OM
  double srr = FAM == kRatA ? srr_a : quad - t2;
  double* sxr = q + 1;  // S_xr[k] = q[1 + k] - sv[1 + k], in place
#pragma unroll
  for (int k = 0; k < NCM; ++k) sxr[k] -= sv[1 + k];
  if constexpr (T > 1) {
#pragma unroll
    for (int k = 0; k < NCM; ++k)
      if (k < M.nc) sxr[k] = lane_sum<T>(sxr[k], mask);
    srr = lane_sum<T>(srr, mask);
    if constexpr (FAM == kSeasonal) {
      sr_tot = lane_sum<T>(sr_tot, mask);
    } else {
      G.a0 = lane_sum<T>(G.a0, mask);
      G.a1 = lane_sum<T>(G.a1, mask);
      if constexpr (FAM == kRadon || FAM == kRatA) G.a2 = lane_sum<T>(G.a2, mask);
      if constexpr (FAM == kRatA) G.a3 = lane_sum<T>(G.a3, mask);
      if (kind == 1) dk0 = lane_sum<T>(dk0, mask);
      if (last) dk1 = lane_sum<T>(dk1, mask);
    }
    if constexpr (FAM != kRatA) sr_all = lane_sum<T>(sr_all, mask);
  }
  if constexpr (FAM != kRatA) {
#pragma unroll
    for (int k = 0; k < NCM; ++k) sxr[k] += M.su[1 + k] * sr_all;  // sum x r = sum x' r + xbar sum r
  }
  k0g += dk0;
  k1g += dk1;
  bool poison = false;
  if (VALUE && fold < M.K) {
    if constexpr (T > 1) __syncwarp(mask);  // group positions stored by their owning lanes
    const int t0 = __ldg(M.sex_lo + fold), t1 = __ldg(M.sex_hi + fold);
    for (int tt = t0 + t; tt < t1; tt += T) {
      const int i = __ldg(M.sex_rows + tt);
      double off = P.off0;
      if constexpr (FAM != kSeasonal) {
        const size_t gi = static_cast<size_t>(__ldg(M.sex_grp + tt)) * nch + c;
        off = group_offset<FAM, NCM>(P, S.pos[(kind == 0 ? cur : cur ^ 1) * plane + gi]);
      }
      double m = off;
      if constexpr (FAM == kRatA) {  // the subject's own slope
        const size_t si = static_cast<size_t>(M.J + __ldg(M.sex_grp + tt)) * nch + c;
        m = fma(S.pos[(kind == 0 ? cur : cur ^ 1) * plane + si], __ldg(M.x + i), off);
      } else {
#pragma unroll
        for (int k = 0; k < NCM; ++k)
          if (k < M.nc) m = fma(P.w[k], __ldg(M.x + static_cast<size_t>(k) * M.n + i), m);
      }
      const double r = __ldg(M.y + i) - m;
      poison |= !isfinite(P.logv + r * r * P.inv_v);
    }
    if constexpr (T > 1) poison = __ballot_sync(mask, poison) != 0;
  }
  bad = T > 1 ? __any_sync(mask, bad) : bad;
  global_grad<FAM, NCM, NGM, true>(M, P, qG, sxr, sr_tot, srr, G, n_train, gG, VALUE, lp);
  if (VALUE && poison) lp = CUDART_NAN;
  if constexpr (T > 1) __syncwarp(mask);
}


// Row-tile ring of the group-batched kernel: the CTA's warps (one chain each) share one staged copy
// of every batch row tile. Tile g of the launch's sequence (pass-major, M.ntile tiles per pass)
// lives in slot g & 1 as [y: rt*32][x: nc][rt*32][key: rt*32]; TMA bulk copies fill it (full[]
// mbarrier), the last of the CTA's W warps to release a tile refills its slot with tile g + 2.
constexpr int kRing = 3;  // ring depth (slots)

// Bytes of one ring slot: y and nc covariate columns of rt rows x 32 lanes, plus the keys unless
// they are group-uniform (0 when the ring is off).
__host__ __device__ inline size_t ring_slot_bytes(const ModelDev& M) {
  if (!M.ring) return 0;
  return static_cast<size_t>(M.rt) * 32 * (8 + 8 * M.nc + (M.bkey_uniform ? 0 : 4));
}

struct BatchRing {
  unsigned char* base;
  size_t slot_bytes;
  unsigned long long* full;
  unsigned int* rel;
  uint32_t g;       // next tile of this warp
  uint32_t total;   // tiles consumed by this launch
  unsigned int W;   // valid warps of the CTA
  double* qslots;   // [2 or 4][nb][kBlock] group position / momentum slots (rat M_A: + slopes)
};

__device__ __forceinline__ void ring_issue(const ModelDev& M, BatchRing& rg, uint32_t g) {
  using namespace tc;
  const int s = g % kRing;
  const int tl = static_cast<int>(g % static_cast<uint32_t>(M.ntile));
  const int r0 = __ldg(M.tile_r0 + tl), rows = __ldg(M.tile_rows + tl);
  const size_t tot = static_cast<size_t>(M.bstride) * 32;
  const uint32_t yb = rows * 32 * 8;
  fence_proxy_async();
  mbar_expect_tx(&rg.full[s], yb * (1 + M.nc) + (M.bkey_uniform ? 0 : rows * 32 * 4));
  unsigned char* dst = rg.base + s * rg.slot_bytes;
  bulk_g2s(dst, M.yb + static_cast<size_t>(r0) * 32, yb, &rg.full[s]);
  for (int k = 0; k < M.nc; ++k)
    bulk_g2s(dst + static_cast<size_t>(M.rt) * 32 * 8 * (1 + k), M.xb + k * tot + static_cast<size_t>(r0) * 32,
             yb, &rg.full[s]);
  if (!M.bkey_uniform)
    bulk_g2s(dst + static_cast<size_t>(M.rt) * 32 * 8 * (1 + M.nc), M.keyb + static_cast<size_t>(r0) * 32,
             rows * 32 * 4, &rg.full[s]);
}

// Rows of one staged tile for one lane (its group, offset `off`). KEYS: 0 = per-row fold keys,
// 1 = group-uniform key and equal group lengths in the batch (no per-row test at all),
// 2 = group-uniform key, rows past the group's end masked by count. NCX: exact covariate count
// (0 = M.nc at run time, up to NCM). Two interleaved partial sums per accumulator.
template <int FAM, int NCX, int NCM, int KEYS, bool VALUE>
__device__ __forceinline__ void tile_rows_loop(const ModelDev& M, const Prep<NCM>& P, const double* yp,
                                               const double* xp, const int* kp, int xstride, int rows,
                                               int jb0, int grows, bool gtrain, int gkey, int lo, int hi,
                                               double off, double& srg, double* sxr, double& srr,
                                               double& srg1, double* sxr1, double& srr1, bool& poison) {
  constexpr int kNc = NCX > 0 ? NCX : NCM;
  const int nc = NCX > 0 ? NCX : M.nc;
  auto row = [&](const double* yq, const double* xq, const int* kq, int jb, double& a_rg, double* a_xr,
                 double& a_rr) {
    double m = off;
    double xs[kNc];
#pragma unroll
    for (int k = 0; k < kNc; ++k) {
      xs[k] = (NCX > 0 || k < nc) ? xq[k * xstride] : 0.0;
      m = fma(P.w[k], xs[k], m);
    }
    const double r = *yq - m;
    bool train, test;
    if constexpr (KEYS == 0) {
      const int ki = *kq;  // padding rows (key < 0) neither train nor test
      train = ki >= 0 && static_cast<unsigned>(ki - lo) >= static_cast<unsigned>(hi - lo);
      test = ki >= 0 && !train;
    } else if constexpr (KEYS == 1) {
      train = gtrain;
      test = gkey >= 0 && !gtrain;
    } else {
      const bool in = jb < grows;
      train = gtrain && in;
      test = gkey >= 0 && !gtrain && in;
    }
    if (train) {
      a_rg += r;
#pragma unroll
      for (int k = 0; k < kNc; ++k) a_xr[k] = fma(xs[k], r, a_xr[k]);
      a_rr = fma(r, r, a_rr);
    }
    if (VALUE && test) poison |= !isfinite(P.logv + r * r * P.inv_v);
  };
  int j = 0;
#pragma unroll 4
  for (; j + 1 < rows; j += 2, yp += 64, xp += 64, kp += 64) {
    row(yp, xp, kp, jb0 + j, srg, sxr, srr);
    row(yp + 32, xp + 32, kp + 32, jb0 + j + 1, srg1, sxr1, srr1);
  }
  if (j < rows) row(yp, xp, kp, jb0 + j, srg, sxr, srr);
}

// Group-batched gradient pass for the hierarchical families (grouped J > 1, radon), one warp per
// chain: lane i owns group slot b of every batch (M.bgroup[b*32 + i], groups sorted by size so a
// batch's groups have similar row counts) and keeps that group's position / momentum in registers
// (qb[b * kBlock], pb[b * kBlock]: per-thread shared-memory slots) across the n_lf passes of a transition. Rows come from the lane-interleaved batch
// layout (M.yb/xb/keyb: row j of batch b for lane i at (boff[b] + j) * 32 + i), so every row step
// is one coalesced warp load and no per-group reduction is needed; only the global sums are
// butterfly-reduced once per pass. Same semantics as grad_pass (kinds 0/1/2); k0g / k1g / bad
// are warp-reduced here so every lane leaves with identical values.
template <int FAM, int NB, int NCM, int NGM, bool VALUE, int NCX>
__device__ __forceinline__ void hgrad_pass(const ModelDev& M, const ChainsDev& S, int c, int t,
                                           int lo, int hi, int n_train, const double* qG, int kind,
                                           bool last, double scale, int cur, NormalCursor& nc,
                                           ChainRng& R, const double* probe_p, double* gG, double& lp,
                                           double& k0g, double& k1g, bool& bad, double* qb,
                                           double* pb, BatchRing& rg) {
  constexpr unsigned kFull = 0xffffffffu;
  Prep<NCM> P;
  prepare<FAM, NCM, NGM>(M, qG, P);
  const int nch = S.nch;
  const double eps = M.step, half = 0.5 * M.step;
  const size_t plane = static_cast<size_t>(M.dim) * nch;
  double sxr[NCM];
#pragma unroll
  for (int k = 0; k < NCM; ++k) sxr[k] = 0.0;
  double srr = 0.0, k0l = 0.0, k1l = 0.0;
  bool poison = false, badl = false;
  GroupAcc G{0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
  for (int b = 0; b < M.nb; ++b) {
    const int g = __ldg(M.bgroup + b * 32 + t);
    const bool valid = g >= 0;
    double qg = 0.0;
    if (valid) {
      const size_t gi = static_cast<size_t>(g) * nch + c;
      const double mg = __ldg(M.inv_mass + g);
      if (kind == 0) {
        qg = S.pos[cur * plane + gi];
      } else if (kind == 1) {
        const double p0 = probe_p ? probe_p[static_cast<size_t>(c) * M.dim + g] : nc.at(R, g) / sqrt(mg);
        k0l += mg * p0 * p0;
        pb[b * kBlock] = p0 + half * S.grad[cur * plane + gi];
        qg = S.pos[cur * plane + gi] + eps * mg * pb[b * kBlock];
      } else {
        qg = qb[b * kBlock] + eps * mg * pb[b * kBlock];
      }
      badl |= !isfinite(qg);
      qb[b * kBlock] = qg;
    }
    // rat M_A: the subject's slope beta_g (dim J + g) is a second group parameter, slots qb2/pb2
    double qs = 0.0;
    double* qb2 = qb + 2 * static_cast<size_t>(M.nb) * kBlock;
    double* pb2 = pb + 2 * static_cast<size_t>(M.nb) * kBlock;
    if constexpr (FAM == kRatA) {
      if (valid) {
        const int gs = M.J + g;
        const size_t si = static_cast<size_t>(gs) * nch + c;
        const double ms = __ldg(M.inv_mass + gs);
        if (kind == 0) {
          qs = S.pos[cur * plane + si];
        } else if (kind == 1) {
          const double p0 = probe_p ? probe_p[static_cast<size_t>(c) * M.dim + gs] : nc.at(R, gs) / sqrt(ms);
          k0l += ms * p0 * p0;
          pb2[b * kBlock] = p0 + half * S.grad[cur * plane + si];
          qs = S.pos[cur * plane + si] + eps * ms * pb2[b * kBlock];
        } else {
          qs = qb2[b * kBlock] + eps * ms * pb2[b * kBlock];
        }
        badl |= !isfinite(qs);
        qb2[b * kBlock] = qs;
      }
    }
    Prep<NCM> Pg = P;  // the row predictor: rat M_A uses the subject's own slope
    if constexpr (FAM == kRatA) Pg.w[0] = qs;
    double sxg[NCM];   // rat M_A: per-subject sum t r (-> d/d beta_g) instead of the global sum
#pragma unroll
    for (int k = 0; k < NCM; ++k) sxg[k] = 0.0;
    double* sxr_tgt = FAM == kRatA ? sxg : sxr;
    const double off = group_offset<FAM, NCM>(P, qg);
    double srg = 0.0, srg1 = 0.0, srr1 = 0.0;
    double sxr1[NCM];
#pragma unroll
    for (int k = 0; k < NCM; ++k) sxr1[k] = 0.0;
    // group-uniform fold keys (e.g. LOGO): one train test per group, rows past the group's end
    // (batch padding) masked by count instead of a per-row key
    const int gkey = __ldg(M.bkey + b * 32 + t);
    const int grows = __ldg(M.bgrows + b * 32 + t);
    const bool gtrain = gkey >= 0 && static_cast<unsigned>(gkey - lo) >= static_cast<unsigned>(hi - lo);
    const int tl1 = __ldg(M.tile_first + b + 1);
    const int bstart = __ldg(M.boff + b);
    for (int tl = __ldg(M.tile_first + b); tl < tl1; ++tl) {
    const int s = rg.g % kRing;
    const int rows = __ldg(M.tile_rows + tl);
    const int tr0 = __ldg(M.tile_r0 + tl);
    const int jb0 = tr0 - bstart;  // row of the batch at tile row 0
    const double* yp;
    const double* xp;
    const int* kp;
    int xstride;
    if (M.ring) {  // staged tile in shared memory
      tc::mbar_wait(&rg.full[s], (rg.g / kRing) & 1u);
      yp = reinterpret_cast<const double*>(rg.base + s * rg.slot_bytes) + t;
      xstride = M.rt * 32;
      xp = yp + xstride;
      kp = reinterpret_cast<const int*>(yp - t + static_cast<size_t>(xstride) * (1 + M.nc)) + t;
    } else {  // straight from L2 / L1 (read-only path)
      yp = M.yb + static_cast<size_t>(tr0) * 32 + t;
      xstride = M.bstride * 32;
      xp = M.xb + static_cast<size_t>(tr0) * 32 + t;
      kp = M.keyb + static_cast<size_t>(tr0) * 32 + t;
    }
    if (M.bkey_uniform) {
      // group-uniform keys: one train flag per group; rows past the group's end only in batches
      // whose groups differ in length (buniform[b] == 0)
      if (__ldg(M.buniform + b))
        tile_rows_loop<FAM, NCX, NCM, 1, VALUE>(M, Pg, yp, xp, kp, xstride, rows, jb0, grows, gtrain, gkey,
                                               lo, hi, off, srg, sxr_tgt, srr, srg1, sxr1, srr1, poison);
      else
        tile_rows_loop<FAM, NCX, NCM, 2, VALUE>(M, Pg, yp, xp, kp, xstride, rows, jb0, grows, gtrain, gkey,
                                               lo, hi, off, srg, sxr_tgt, srr, srg1, sxr1, srr1, poison);
    } else {
      tile_rows_loop<FAM, NCX, NCM, 0, VALUE>(M, Pg, yp, xp, kp, xstride, rows, jb0, grows, gtrain, gkey,
                                             lo, hi, off, srg, sxr_tgt, srr, srg1, sxr1, srr1, poison);
    }
    if (M.ring) {
    __syncwarp(kFull);
    if (t == 0) {  // release the slot; the CTA's last warp refills it
      const unsigned int old = atomicAdd(&rg.rel[s], 1u);
      if ((old + 1u) % rg.W == 0u && rg.g + kRing < rg.total) ring_issue(M, rg, rg.g + kRing);
    }
    ++rg.g;
    }
    }
    srg += srg1;
    srr += srr1;
#pragma unroll
    for (int k = 0; k < NCM; ++k) sxr_tgt[k] += sxr1[k];
    if constexpr (FAM == kRatA) {  // slope beta_g: t r / vy - (beta_g - mu_b) / vb (rat_growth.cpp:127-137)
      if (valid) {
        const int gs = M.J + g;
        const size_t si = static_cast<size_t>(gs) * nch + c;
        const double db = qs - qG[1];
        G.a2 += db / P.vb;
        G.a3 += db * db;
        const double gsl = sxg[0] / P.v - db / P.vb;
        badl |= !isfinite(gsl);
        if (kind == 0) {
          S.grad[cur * plane + si] = gsl;
        } else {
          const double pn = pb2[b * kBlock] + scale * gsl;
          pb2[b * kBlock] = pn;
          badl |= !isfinite(pn);
          if (last) {
            S.pos[(cur ^ 1) * plane + si] = qs;
            S.grad[(cur ^ 1) * plane + si] = gsl;
            k1l += __ldg(M.inv_mass + gs) * pn * pn;
            if (probe_p && S.probe_p_out) S.probe_p_out[static_cast<size_t>(c) * M.dim + gs] = pn;
          }
        }
      }
    }
    if (valid) {
      const double gg = group_grad<FAM, NCM, NGM>(P, qG, M, qg, srg, G);
      const size_t gi = static_cast<size_t>(g) * nch + c;
      badl |= !isfinite(gg);
      if (kind == 0) {
        S.grad[cur * plane + gi] = gg;
      } else {
        const double pn = pb[b * kBlock] + scale * gg;
        pb[b * kBlock] = pn;
        badl |= !isfinite(pn);
        if (last) {
          S.pos[(cur ^ 1) * plane + gi] = qg;
          S.grad[(cur ^ 1) * plane + gi] = gg;
          k1l += __ldg(M.inv_mass + g) * pn * pn;
          if (probe_p && S.probe_p_out) S.probe_p_out[static_cast<size_t>(c) * M.dim + g] = pn;
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NCM; ++k) sxr[k] = lane_sum<32>(sxr[k], kFull);
  srr = lane_sum<32>(srr, kFull);
  G.a0 = lane_sum<32>(G.a0, kFull);
  G.a1 = lane_sum<32>(G.a1, kFull);
  G.a2 = lane_sum<32>(G.a2, kFull);
  G.a3 = lane_sum<32>(G.a3, kFull);
  if (kind == 1) k0g += lane_sum<32>(k0l, kFull);
  if (last) k1g += lane_sum<32>(k1l, kFull);
  bad |= __any_sync(kFull, badl);
  if (VALUE) poison = __any_sync(kFull, poison);
  global_grad<FAM, NCM, NGM>(M, P, qG, sxr, 0.0, srr, G, n_train, gG, VALUE, lp);
  if (VALUE && poison) lp = CUDART_NAN;
  __syncwarp(kFull);  // group-dim stores become visible to the chain's lanes
}

// Unseen subject of the per-subject-slope growth model: log N(y; mu_a + mu_b t, va + vb t t' +
// vy I) by a dense Cholesky (mvn_logpdf_chol, math.hpp:46-90); -inf when not positive definite.
// Subjects have at most kRatMaxObs rows on device (checked at upload).
constexpr int kRatMaxObs = 16;
__device__ double rat_unseen_logpdf(const ModelDev& M, int r0, int r1, double mu_a, double mu_b,
                                    double va, double vb, double vy) {
  const int n = r1 - r0;
  double L[kRatMaxObs * (kRatMaxObs + 1) / 2], tv[kRatMaxObs], r[kRatMaxObs];
  for (int a = 0; a < n; ++a) {
    const int i = __ldg(M.seg_rows + r0 + a);
    tv[a] = __ldg(M.x + i);
    r[a] = __ldg(M.y + i) - (mu_a + mu_b * tv[a]);
  }
  for (int j = 0; j < n; ++j) {  // packed lower triangle, row i at i(i+1)/2
    double d = va + vb * tv[j] * tv[j] + vy;
    for (int k = 0; k < j; ++k) d -= L[j * (j + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
    if (!(d > 0.0) || !isfinite(d)) return -CUDART_INF;
    const double l = sqrt(d);
    L[j * (j + 1) / 2 + j] = l;
    for (int i = j + 1; i < n; ++i) {
      double sm = va + vb * tv[i] * tv[j];
      for (int k = 0; k < j; ++k) sm -= L[i * (i + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
      L[i * (i + 1) / 2 + j] = sm / l;
    }
  }
  double q = 0.0, ld = 0.0;
  for (int i = 0; i < n; ++i) {
    double sm = r[i];
    for (int k = 0; k < i; ++k) sm -= L[i * (i + 1) / 2 + k] * r[k];
    r[i] = sm / L[i * (i + 1) / 2 + i];
    q += r[i] * r[i];
    ld += log(L[i * (i + 1) / 2 + i]);
  }
  return -0.5 * (n * kLog2Pi + 2.0 * ld + q);
}

// Model::log_pred at the stored position (grouped_regression.cpp:124-163, radon.cpp:109-138,
// seasonal_ar.cpp:107-115), observations split across the chain's lanes.
template <int FAM, int T, int NCM, int NGM>
__device__ double log_pred(const ModelDev& M, const ChainsDev& S, int c, int t, unsigned mask,
                           int fold, int cur, const double* qG) {
  if (fold >= M.K) return 0.0;
  Prep<NCM> P;
  prepare<FAM, NCM, NGM>(M, qG, P);
  const size_t plane = static_cast<size_t>(M.dim) * S.nch;
  const int s0 = __ldg(M.fold_seg + fold), s1 = __ldg(M.fold_seg + fold + 1);
  double v_pred = P.v, va_pred = P.va, vb_pred = 0.0;
  if constexpr (FAM == kSeasonal) v_pred = exp(2.0 * qG[1]);
  if constexpr (FAM == kRatB) {  // rat_growth.cpp:204-205 (exp(2 theta) forms)
    va_pred = exp(2.0 * qG[2]);
    v_pred = exp(2.0 * qG[3]);
  }
  if constexpr (FAM == kRatA) {  // rat_growth.cpp:181-183
    va_pred = exp(2.0 * qG[2]);
    vb_pred = exp(2.0 * qG[3]);
    v_pred = exp(2.0 * qG[4]);
  }
  double lp = 0.0;
  for (int s = s0; s < s1; ++s) {
    const int r0 = __ldg(M.seg_row + s), r1 = __ldg(M.seg_row + s + 1);
    const int g = __ldg(M.seg_group + s);
    const bool unseen = __ldg(M.seg_unseen + s) != 0;
    double qg = 0.0;
    if (FAM != kSeasonal && !unseen) qg = S.pos[cur * plane + static_cast<size_t>(g) * S.nch + c];
    if constexpr (FAM == kRatA) {
      if (unseen) {  // dense N(mu_a + mu_b t, va + vb t t' + vy I) over the subject (rat_growth.cpp:184-199)
        double part = 0.0;
        if (t == 0) part = rat_unseen_logpdf(M, r0, r1, qG[0], qG[1], va_pred, vb_pred, v_pred);
        lp += lane_sum<T>(part, mask);
        continue;
      }
      P.w[0] = S.pos[cur * plane + static_cast<size_t>(M.J + g) * S.nch + c];  // the subject's slope
    }
    double a = 0.0, b = 0.0;
    for (int tt = r0 + t; tt < r1; tt += T) {
      const int i = __ldg(M.seg_rows + tt);
      double m;
      if constexpr (FAM == kGrouped) m = unseen ? qG[0] : qg;
      else if constexpr (FAM == kRadon) m = unseen ? P.off0 : P.off0 + sqrt(P.va) * qg;
      else if constexpr (FAM == kRatB) m = unseen ? qG[1] : qg;
      else if constexpr (FAM == kRatA) m = qg;
      else m = P.off0;
#pragma unroll
      for (int k = 0; k < NCM; ++k)
        if (k < M.nc) m = fma(P.w[k], __ldg(M.x + static_cast<size_t>(k) * M.n + i), m);
      const double r = __ldg(M.y + i) - m;
      if (unseen) {
        a += r * r;
        b += r;
      } else {
        a += -0.5 * (kLog2Pi + log(v_pred) + r * r / v_pred);
      }
    }
    a = lane_sum<T>(a, mask);
    if (unseen) {  // mvn_logpdf_compound, math.hpp:94-109, sigma2 = vy, tau2 = va
      b = lane_sum<T>(b, mask);
      const double sigma2 = FAM == kRatB ? v_pred : P.v, tau2 = FAM == kRatB ? va_pred : P.va;
      const int nn = r1 - r0;
      if (!(sigma2 > 0.0) || tau2 < 0.0) return CUDART_NAN;  // numeric_fault in the reference
      const double denom = sigma2 + nn * tau2;
      const double quad = (a - tau2 * b * b / denom) / sigma2;
      const double logdet = (nn - 1) * log(sigma2) + log(denom);
      lp += -0.5 * (nn * kLog2Pi + logdet + quad);
    } else {
      lp += a;
    }
  }
  return lp;
}

// HS / DSS state after hmc_step + log_pred (engine.cpp:360-373; warm-up hmc.cpp:133-145):
// pred_derivs / pred_sample of grouped_regression.cpp:190-213, radon.cpp:167-199 and
// seasonal_ar.cpp:133-150 over the fold's test rows in fold_meta order. The lanes of the chain
// split the rows; DSS draws come from the chain stream in row order on every lane (so all lanes
// keep identical stream state), the lane owning row t uses normal t.
template <int FAM, int T, int NCM, int NGM>
__device__ void score_extra(const ModelDev& M, const ChainsDev& S, int c, int t, unsigned mask,
                            int fold, int cur, const double* qG, bool warm, ChainRng& R) {
  const ExtraDev& X = S.X;
  const int L = S.L, kf = fold - S.fold0, cl = c % L;
  Prep<NCM> P;
  prepare<FAM, NCM, NGM>(M, qG, P);
  double vy, sy, sa = 0.0;
  if constexpr (FAM == kGrouped) {
    sy = exp(qG[2]);  // sig_y
    vy = sy * sy;
  } else if constexpr (FAM == kRatA || FAM == kRatB) {  // rat_growth.cpp:267-290
    sy = exp(qG[NGM - 1]);
    vy = sy * sy;
  } else if constexpr (FAM == kRadon) {
    vy = exp(qG[3]);
    sy = exp(0.5 * qG[3]);
    sa = exp(0.5 * qG[2]);
  } else {
    vy = exp(2.0 * qG[1]);
    sy = exp(qG[1]);
  }
  const size_t plane = static_cast<size_t>(M.dim) * S.nch;
  const int s0 = __ldg(M.fold_seg + fold), s1 = __ldg(M.fold_seg + fold + 1);
  int rt = 0;
  for (int s = s0; s < s1; ++s) {
    const int r0 = __ldg(M.seg_row + s), r1 = __ldg(M.seg_row + s + 1);
    double qg = 0.0;
    if constexpr (FAM != kSeasonal) qg = S.pos[cur * plane + static_cast<size_t>(__ldg(M.seg_group + s)) * S.nch + c];
    for (int tt = r0; tt < r1; ++tt, ++rt) {
      const double z = X.kind == 2 ? R.normal() : 0.0;
      if (rt % T != t) continue;
      const int i = __ldg(M.seg_rows + tt);
      double mean;
      if constexpr (FAM == kRadon) {
        mean = qG[1] + sa * qg + (M.include_floor ? 1.0 : 0.0) * qG[0] * __ldg(M.x + i);
      } else if constexpr (FAM == kRatA) {
        const double slope = S.pos[cur * plane + static_cast<size_t>(M.J + __ldg(M.seg_group + s)) * S.nch + c];
        mean = fma(slope, __ldg(M.x + i), qg);
      } else {
        mean = (FAM == kGrouped || FAM == kRatB) ? qg : P.off0;
#pragma unroll
        for (int k = 0; k < NCM; ++k)
          if (k < M.nc) mean = fma(P.w[k], __ldg(M.x + static_cast<size_t>(k) * M.n + i), mean);
      }
      if (X.kind == 1) {
        const double d1 = -(__ldg(M.y + i) - mean) / vy;
        extra_hs_row(X, kf, cl, L, rt, d1, -1.0 / vy, warm);
      } else {
        extra_dss_row(X, kf, cl, L, rt, mean + sy * z, warm);
      }
    }
  }
  if (X.kind == 2 && !warm) {
    __syncwarp(mask);  // staged deviations of every lane's rows
    extra_dss_cov(X, kf, cl, L, t, T);
  }
}

// NB = 0: row-split passes (grad_pass, T lanes per chain); NB > 0: group-batched passes
// (hgrad_pass, T = 32, up to 32 * NB groups).
template <int FAM, int T, int NCM, int NGM, int NB>
__global__ void __launch_bounds__(kBlock, NB > 0 ? 3 : (NB == -2 ? 4 : (NB < 0 && T > 1 ? 4 : 1))) gauss_kernel(ModelDev M, ChainsDev S, RunArgs A) {
  constexpr int kChains = kBlock / T;
  const int t = threadIdx.x % T;
  const int local = threadIdx.x / T;
  const int c = blockIdx.x * kChains + local;
  BatchRing rg{};
  if constexpr (NB > 0) {
    extern __shared__ __align__(128) unsigned char ring_raw[];
    const size_t slot_bytes = ring_slot_bytes(M);
    rg.base = ring_raw;
    rg.slot_bytes = slot_bytes;
    rg.full = reinterpret_cast<unsigned long long*>(ring_raw + kRing * slot_bytes);
    rg.rel = reinterpret_cast<unsigned int*>(rg.full + kRing);
    rg.qslots = reinterpret_cast<double*>(ring_raw + kRing * slot_bytes + 16 * kRing);
    rg.g = 0;
    const uint32_t passes = A.mode == kModeEval ? 1u : (A.mode == kModePred ? 0u : static_cast<uint32_t>(A.n_iters * M.n_lf));
    rg.total = M.ring ? passes * static_cast<uint32_t>(M.ntile) : 0u;
    rg.W = static_cast<unsigned int>(min(kChains, S.nch - static_cast<int>(blockIdx.x) * kChains));
    if (threadIdx.x < kRing) {
      tc::mbar_init(&rg.full[threadIdx.x], 1);
      rg.rel[threadIdx.x] = 0u;
    }
    tc::fence_mbar_init();
    __syncthreads();
    if (threadIdx.x == 0)
      for (uint32_t g = 0; g < kRing && g < rg.total; ++g) ring_issue(M, rg, g);
  }
  if (c >= S.nch) return;
  const unsigned mask =
      T == 32 ? 0xffffffffu : (((1u << T) - 1u) << ((threadIdx.x & 31) & ~(T - 1)));
  const int nch = S.nch;
  const int fold = S.fold_override ? S.fold_override[c] : S.fold0 + c / S.L;
  const int lo = __ldg(M.fold_lo + fold), hi = __ldg(M.fold_hi + fold);
  const int n_train = __ldg(M.n_train + fold);
  const int J = M.J, ng = M.ng;
  const size_t plane = static_cast<size_t>(M.dim) * nch;
  // address of global parameter slot i of chain c in plane b
  auto gaddr = [&](int b, int i) { return b * plane + static_cast<size_t>(M.goff + gidx<FAM>(M, i)) * nch + c; };
  int cur = S.cur[c];

  double qG[NGM], pG[NGM], gG[NGM];
#pragma unroll
  for (int i = 0; i < NGM; ++i) {
    qG[i] = i < ng ? S.pos[gaddr(cur, i)] : 0.0;
    gG[i] = 0.0;
  }
  double lp0 = S.lp0[c];
  ChainRng R;
  R.init(S.seed, S.rng_stream[c], S.rng_pos[c], S.rng_cached[c], S.rng_has[c] != 0);
  NormalCursor nc;
  constexpr int kNB = 1;
  constexpr int NCX = NB > 0 ? NB - 1 : 0;  // exact covariate count of the batched variant (0 = run time)
  // group slots of each thread (NB > 0): [nb][kBlock] position / momentum after the ring
  double* qb = rg.qslots + threadIdx.x;
  double* pb = rg.qslots + static_cast<size_t>(M.nb) * kBlock + threadIdx.x;
  // group slots of each thread (NB < 0, suff_slots): [ns][kBlock] position, then momentum
  double* sq = nullptr;
  double* sp = nullptr;
  if constexpr (NB < 0) {
    extern __shared__ __align__(16) double suff_raw[];
    const int ns = suff_slots(M, T);
    if (ns > 0) {
      sq = suff_raw + threadIdx.x;
      sp = suff_raw + static_cast<size_t>(ns) * kBlock + threadIdx.x;
    }
  }

  if (A.mode == kModeEval || A.mode == kModePred) {
    if (A.mode == kModeEval) {
      double lp = 0.0, k0 = 0.0, k1 = 0.0;
      bool bad = false;
      if constexpr (NB > 0)
        hgrad_pass<FAM, kNB, NCM, NGM, true, NCX>(M, S, c, t, lo, hi, n_train, qG, 0, false, 0.0, cur, nc,
                                             R, nullptr, gG, lp, k0, k1, bad, qb, pb, rg);
      else if constexpr (NB < 0)
        suff_pass<FAM, T, NCM, NGM, true>(M, S, c, t, mask, fold, n_train, qG, 0, false, 0.0, cur, nc, R,
                                          nullptr, gG, lp, k0, k1, bad, nullptr, nullptr);
      else
        grad_pass<FAM, T, NCM, NGM, true>(M, S, c, t, mask, lo, hi, n_train, qG, 0, false, 0.0,
                                          cur, nc, R, nullptr, gG, lp, k0, k1, bad);
      if (t == 0) {
#pragma unroll
        for (int i = 0; i < NGM; ++i)
          if (i < ng) S.grad[gaddr(cur, i)] = gG[i];
        S.lp0[c] = lp;
        if (A.out_a) A.out_a[c] = lp;
      }
    } else {
      const double s = log_pred<FAM, T, NCM, NGM>(M, S, c, t, mask, fold, cur, qG);
      if (t == 0 && A.out_a) A.out_a[c] = s;
    }
    return;
  }

  const double eps = M.step, half = 0.5 * M.step;
  const int n_lf = M.n_lf;
  int64_t div_count = 0;
  double warm = 0.0;
  for (int64_t it = 0; it < A.n_iters; ++it) {
    const double* probe_p = A.mode == kModeProbe ? A.probe_momentum : nullptr;
    nc.start(R);
    // Momentum refresh of the global dims (normals J..dim-1 of this transition) + half kick.
    double k0G = 0.0;
#pragma unroll
    for (int i = 0; i < NGM; ++i) {
      if (i < ng) {
        const int gi = M.goff + gidx<FAM>(M, i);
        const double mi = __ldg(M.inv_mass + gi);
        const double p0 = probe_p ? probe_p[static_cast<size_t>(c) * M.dim + gi]
                                  : nc.at(R, gi) / sqrt(mi);
        k0G += mi * p0 * p0;
        pG[i] = p0 + half * S.grad[gaddr(cur, i)];
      }
    }
    bool bad = false;
    double lp1 = 0.0, k0g = 0.0, k1g = 0.0;
    for (int s = 0; s < n_lf; ++s) {
      const bool first = s == 0, last = s == n_lf - 1;
#pragma unroll
      for (int i = 0; i < NGM; ++i) {
        if (i < ng) {
          const double base = first ? S.pos[gaddr(cur, i)] : qG[i];
          qG[i] = base + eps * __ldg(M.inv_mass + M.goff + gidx<FAM>(M, i)) * pG[i];
          bad |= !isfinite(qG[i]);
        } else {
          qG[i] = 0.0;
        }
      }
      const double scale = last ? half : eps;
      if constexpr (NB > 0) {
        if (last)
          hgrad_pass<FAM, kNB, NCM, NGM, true, NCX>(M, S, c, t, lo, hi, n_train, qG, first ? 1 : 2, true,
                                               scale, cur, nc, R, probe_p, gG, lp1, k0g, k1g, bad, qb, pb, rg);
        else
          hgrad_pass<FAM, kNB, NCM, NGM, false, NCX>(M, S, c, t, lo, hi, n_train, qG, first ? 1 : 2, false,
                                                scale, cur, nc, R, probe_p, gG, lp1, k0g, k1g, bad, qb, pb, rg);
      } else if constexpr (NB < 0) {
        // two inlined copies (value / gradient-only): a run-time flag measured 3-15% slower
        if (last)
          suff_pass<FAM, T, NCM, NGM, true>(M, S, c, t, mask, fold, n_train, qG, first ? 1 : 2, true, scale,
                                            cur, nc, R, probe_p, gG, lp1, k0g, k1g, bad, sq, sp);
        else
          suff_pass<FAM, T, NCM, NGM, false>(M, S, c, t, mask, fold, n_train, qG, first ? 1 : 2, false, scale,
                                             cur, nc, R, probe_p, gG, lp1, k0g, k1g, bad, sq, sp);
      } else if (last) {
        grad_pass<FAM, T, NCM, NGM, true>(M, S, c, t, mask, lo, hi, n_train, qG, first ? 1 : 2,
                                          true, scale, cur, nc, R, probe_p, gG, lp1, k0g, k1g, bad);
      } else {
        grad_pass<FAM, T, NCM, NGM, false>(M, S, c, t, mask, lo, hi, n_train, qG, first ? 1 : 2,
                                           false, scale, cur, nc, R, probe_p, gG, lp1, k0g, k1g, bad);
      }
#pragma unroll
      for (int i = 0; i < NGM; ++i) {
        if (i < ng) {
          bad |= !isfinite(gG[i]);
          pG[i] += scale * gG[i];
          bad |= !isfinite(pG[i]);
        }
      }
    }
    if (!probe_p) nc.finish(R, M.dim);
    double k1G = 0.0;
#pragma unroll
    for (int i = 0; i < NGM; ++i)
      if (i < ng) k1G += __ldg(M.inv_mass + M.goff + gidx<FAM>(M, i)) * pG[i] * pG[i];
    // proposal (q', grad(q')) of the global dims into the working plane; accept flips `cur`
    if (t == 0) {
#pragma unroll
      for (int i = 0; i < NGM; ++i) {
        if (i < ng) {
          S.pos[gaddr(cur ^ 1, i)] = qG[i];
          S.grad[gaddr(cur ^ 1, i)] = gG[i];
        }
      }
    }
    bad |= fold == M.broken_fold;
    const double h0 = -lp0 + 0.5 * (k0g + k0G);
    const double h1 = bad ? CUDART_NAN : -lp1 + 0.5 * (k1g + k1G);
    const double dh = h1 - h0;
    const bool divergent = bad || isnan(dh) || (isfinite(dh) && fabs(dh) > 1000.0);
    bool accepted = false;
    if (divergent) {
      ++div_count;
    } else {
      const double u = probe_p ? A.probe_u[c] : R.uniform();
      if (log(u) < -dh) {
        accepted = true;
        cur ^= 1;
        lp0 = lp1;
      }
    }
    __syncwarp(mask);  // lane 0's stores are read by the chain's lanes below / next pass
    if (A.mode == kModeProbe) {
      if (t == 0) {
        A.out_a[c] = h0;
        A.out_b[c] = h1;
        A.out_flags[c] = (accepted ? 1 : 0) | (divergent ? 2 : 0);
        if (A.traj) {  // final momentum of the trajectory (leapfrog probe)
#pragma unroll
          for (int i = 0; i < NGM; ++i)
            if (i < ng) A.traj[static_cast<size_t>(c) * M.dim + M.goff + gidx<FAM>(M, i)] = pG[i];
          if constexpr (NB <= 0)
            for (int g = 0; g < M.goff; ++g) A.traj[static_cast<size_t>(c) * M.dim + g] = S.wp[static_cast<size_t>(g) * nch + c];
        }
      }
      continue;
    }
    if (A.mode == kModeChain) {  // trace: record (it, chain) = it * nch + c
      if (t == 0) {
        const size_t row = static_cast<size_t>(it) * nch + c;
        if (A.traj)
          for (int d = 0; d < M.dim; ++d)
            A.traj[row * M.dim + d] = S.pos[cur * plane + static_cast<size_t>(d) * nch + c];
        if (A.traj_div) A.traj_div[row] = (accepted ? 1 : 0) | (divergent ? 2 : 0);
        if (A.out_a) A.out_a[row] = h0;
        if (A.out_b) A.out_b[row] = h1;
      }
      continue;
    }
#pragma unroll
    for (int i = 0; i < NGM; ++i) qG[i] = i < ng ? S.pos[gaddr(cur, i)] : 0.0;
    const double sp = log_pred<FAM, T, NCM, NGM>(M, S, c, t, mask, fold, cur, qG);
    if (S.X.kind != 0 && fold < M.K)
      score_extra<FAM, T, NCM, NGM>(M, S, c, t, mask, fold, cur, qG, A.mode == kModeWarmup, R);
    if (A.mode == kModeWarmup) {
      warm += sp;
    } else if (t == 0) {
      accum_observe(S.acc, c, nch, sp, A.iter0 + it, A.planned_n, A.D, A.b);
    }
  }
  if (t == 0) {
    S.cur[c] = static_cast<int8_t>(cur);
    S.lp0[c] = lp0;
    S.rng_pos[c] = R.pos;
    S.rng_cached[c] = R.cached;
    S.rng_has[c] = R.has_cached ? 1 : 0;
    S.divergences[c] += div_count;
    if (A.mode == kModeWarmup) S.warm_sum[c] += warm;
  }
}

}  // namespace

}  // namespace pcvg
