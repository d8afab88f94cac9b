// HS / DSS scoring state on device (the non-LogS branches of engine.cpp:322-373, fed after every
// hmc_step + log_pred). Layout in types.cuh (ExtraDev). Every update mirrors the reference
// accumulator arithmetic:
//   HS  xi = (d2 + d1*d1, d1) per test row (engine.cpp:364-368), WelfordDiag::add (accum.cpp:66-74)
//   DSS one pred_sample draw per test row from the chain stream (engine.cpp:371), then
//       WelfordAccumulator::add (accum.cpp:19-26): a_x[i] += x_i - c_i, a_xx[i][j<=i] += d_i d_j
// Warm-up (hmc.cpp:133-145) sums the raw quantities; the centring kernel divides by L * N_wu.
#pragma once
#include "types.cuh"

namespace pcvg {

// Test row t (fold order) of chain cl in local fold kf: HS update from the predictive derivatives.
__device__ __forceinline__ void extra_hs_row(const ExtraDev& X, int kf, int cl, int L, int t,
                                             double d1, double d2, bool warm) {
  const int m = X.msize[kf];
  const double x1 = d2 + d1 * d1, x2 = d1;
  if (warm) {
    double* W = X.warm + X.wbase[kf] + cl;
    W[static_cast<int64_t>(t) * L] += x1;
    W[static_cast<int64_t>(m + t) * L] += x2;
    return;
  }
  const double* C = X.center + X.cbase[kf];
  const double a = x1 - C[t], b = x2 - C[m + t];
  double* A = X.acc + X.base[kf] + cl;
  A[static_cast<int64_t>(t) * L] += a;
  A[static_cast<int64_t>(m + t) * L] += b;
  A[static_cast<int64_t>(2 * m + t) * L] += a * a;
  A[static_cast<int64_t>(3 * m + t) * L] += b * b;
}

// DSS: the predictive draw of test row t. Sampling mode stages d = x - c for the triangle update.
__device__ __forceinline__ void extra_dss_row(const ExtraDev& X, int kf, int cl, int L, int t,
                                              double draw, bool warm) {
  if (warm) {
    X.warm[X.wbase[kf] + static_cast<int64_t>(t) * L + cl] += draw;
    return;
  }
  const double d = draw - X.center[X.cbase[kf] + t];
  X.acc[X.base[kf] + static_cast<int64_t>(t) * L + cl] += d;
  X.dev[X.wbase[kf] + static_cast<int64_t>(t) * L + cl] = d;
}

// DSS: a_xx[i][j] += d_i d_j for j <= i, rows i = lane, lane + nl, ... (the staged d of every row
// must be visible to the calling lanes).
__device__ __forceinline__ void extra_dss_cov(const ExtraDev& X, int kf, int cl, int L, int lane,
                                              int nl) {
  const int m = X.msize[kf];
  const double* D = X.dev + X.wbase[kf] + cl;
  double* A = X.acc + X.base[kf] + static_cast<int64_t>(m) * L + cl;
  for (int i = lane; i < m; i += nl) {
    const double di = D[static_cast<int64_t>(i) * L];
    double* row = A + (static_cast<int64_t>(i) * (i + 1) / 2) * L;
    for (int j = 0; j <= i; ++j) row[static_cast<int64_t>(j) * L] += di * D[static_cast<int64_t>(j) * L];
  }
}

// Entries per chain of the HS / DSS accumulator, warm-up sums and centre for test size m.
__host__ __device__ inline int64_t extra_acc_len(int kind, int64_t m) {
  return kind == 1 ? 4 * m : (kind == 2 ? m + m * (m + 1) / 2 : 0);
}
__host__ __device__ inline int64_t extra_warm_len(int kind, int64_t m) {
  return kind == 1 ? 2 * m : (kind == 2 ? m : 0);
}

}  // namespace pcvg
