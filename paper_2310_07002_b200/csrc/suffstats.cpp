// Fold-masked sufficient statistics of the Gaussian linear families.
//
// Every Gaussian family's per-row term depends on the data only through u_i = (y_i, x_i) and the
// row's group: r_i = y_i - off(g_i) - w.x_i = om.u_i - off(g_i) with om = (1, -w). So the three
// masked sums the gradient and log joint need (grouped_regression.cpp:87-122, radon.cpp:76-107,
// seasonal_ar.cpp:79-105) are linear / quadratic forms in fold statistics:
//   S_r[g]   = om.s_g - n_g off_g                        s_g = sum of u over g's training rows
//   S_xr[c]  = (A om)[1+c] - sum_g off_g s_g[1+c]        A   = sum of u u^T over training rows
//   S_rr     = om^T A om - sum_g off_g (2 om.s_g - n_g off_g)
// The host builds, once per model: A_k for every fold k (and the sentinel K), the full-data group
// statistics, and per fold the statistics of the groups the fold touches. Training sums are
// formed as (full - excluded) in double-double arithmetic and rounded once, so each entry is the
// training-row sum to ~1 ulp whatever the excluded set; a group with no training row gets exact
// zeros. The excluded rows of each fold (key-sorted) are kept so the value pass can reproduce the
// reference's poisoning by a non-finite masked row (grouped_regression.cpp:74-76).
// Centring: the statistics are of u' = u - ubar (ubar the full-data column means), formed from the
// double-double sums as A' = A - ubar s^T - s ubar^T + n ubar ubar^T and s'_g = s_g - n_g ubar before
// the single rounding. With r_i = om.u'_i - (off_g - om.ubar) the kernel's S_rr = om^T A' om - ...
// then cancels only ~eps * sum (u - ubar)^2 / sum r^2 instead of ~eps * sum y^2 / sum r^2, which for
// data with a large level (y ~ 1e4 +- 1) is the difference between 1e-16 and 1e-8 relative error.
// The per-subject Grams of the growth model M_A stay uncentred (ubar = 0).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

#include "suffstats.hpp"

namespace pcvg {

namespace {

struct DD {
  double hi = 0.0, lo = 0.0;
};

// x += a + ae (a, ae: an exact product split or a plain value with ae = 0), Knuth TwoSum.
inline void dd_add(DD& x, double a, double ae) {
  const double s = x.hi + a;
  const double bb = s - x.hi;
  double e = (x.hi - (s - bb)) + (a - bb);
  e += x.lo + ae;
  x.hi = s + e;
  x.lo = e - (x.hi - s);
}

inline void dd_add_prod(DD& x, double a, double b, double sign) {
  const double p = a * b;
  const double pe = std::fma(a, b, -p);
  dd_add(x, sign * p, sign * pe);
}

inline double dd_val(const DD& x) { return x.hi + x.lo; }

}  // namespace

// y[n], xc[nc][n] and key[n] in device row order; grp_ptr[J+1] (group-major rows) or null for
// J = 0 (one pseudo-group holding every row); fold k holds out rows with lo[k] <= key < hi[k].
// Returns false (no statistics) when a data value or a Gram entry is non-finite: full - excluded
// would not give the reference's per-row masking then.
// group_gram: also the per-group Gram of u (the per-subject-slope growth model, whose sums are all
// per subject).
bool build_suffstats(int64_t n, int nc, int J, const double* y, const double* xc, const int* key,
                     const int* grp_ptr, int K, const int* lo, const int* hi, SuffStats& S,
                     bool group_gram, bool center) {
  const int d = nc + 1, dp = d * (d + 1) / 2, Jg = J > 0 ? J : 1;
  for (int64_t i = 0; i < n; ++i) {
    if (!std::isfinite(y[i])) return false;
    for (int c = 0; c < nc; ++c)
      if (!std::isfinite(xc[static_cast<size_t>(c) * n + i])) return false;
  }
  S.d = d;
  S.dp = dp;
  std::vector<int> grp(n, 0);
  if (J > 0)
    for (int g = 0; g < J; ++g)
      for (int r = grp_ptr[g]; r < grp_ptr[g + 1]; ++r) grp[r] = g;
  auto u = [&](int64_t r, int i) { return i == 0 ? y[r] : xc[static_cast<size_t>(i - 1) * n + r]; };

  // full-data statistics
  std::vector<DD> Af(dp), gsf(static_cast<size_t>(Jg) * d), gAf(group_gram ? static_cast<size_t>(Jg) * dp : 0);
  std::vector<int64_t> gnf(Jg, 0);
  for (int64_t r = 0; r < n; ++r) {
    for (int i = 0; i < d; ++i)
      for (int j = 0; j <= i; ++j) dd_add_prod(Af[i * (i + 1) / 2 + j], u(r, i), u(r, j), 1.0);
    const int g = grp[r];
    if (group_gram)
      for (int i = 0; i < d; ++i)
        for (int j = 0; j <= i; ++j)
          dd_add_prod(gAf[static_cast<size_t>(g) * dp + i * (i + 1) / 2 + j], u(r, i), u(r, j), 1.0);
    ++gnf[g];
    for (int i = 0; i < d; ++i) dd_add(gsf[static_cast<size_t>(g) * d + i], u(r, i), 0.0);
  }
  for (const DD& a : Af)
    if (!std::isfinite(a.hi) || !std::isfinite(a.lo)) return false;  // overflowing products
  // the centre and the full-data sum of u (over all groups)
  std::vector<DD> sf(d);
  for (int g = 0; g < Jg; ++g)
    for (int i = 0; i < d; ++i) {
      const DD& v = gsf[static_cast<size_t>(g) * d + i];
      dd_add(sf[i], v.hi, v.lo);
    }
  S.ubar.assign(d, 0.0);
  if (center && !group_gram && n > 0)
    for (int i = 0; i < d; ++i) S.ubar[i] = dd_val(sf[i]) / static_cast<double>(n);
  const std::vector<double>& ub = S.ubar;
  // s' = s - cnt ubar, rounded once
  auto centred_sum = [&](const DD& v, double cnt, int i) {
    DD x = v;
    dd_add_prod(x, cnt, ub[i], -1.0);
    return dd_val(x);
  };
  S.gn.resize(Jg);
  S.gs.resize(static_cast<size_t>(Jg) * d);
  for (int g = 0; g < Jg; ++g) {
    S.gn[g] = static_cast<double>(gnf[g]);
    for (int i = 0; i < d; ++i)
      S.gs[static_cast<size_t>(g) * d + i] = centred_sum(gsf[static_cast<size_t>(g) * d + i], static_cast<double>(gnf[g]), i);
  }
  S.gA.resize(gAf.size());
  for (size_t i = 0; i < gAf.size(); ++i) S.gA[i] = dd_val(gAf[i]);

  // rows in key order: a fold's excluded rows are one contiguous run
  S.ex_rows.resize(n);
  std::iota(S.ex_rows.begin(), S.ex_rows.end(), 0);
  std::stable_sort(S.ex_rows.begin(), S.ex_rows.end(), [&](int a, int b) { return key[a] < key[b]; });
  S.ex_grp.resize(n);
  std::vector<int> skey(n);
  for (int64_t t = 0; t < n; ++t) {
    S.ex_grp[t] = grp[S.ex_rows[t]];
    skey[t] = key[S.ex_rows[t]];
  }
  S.ex_lo.assign(K + 1, 0);
  S.ex_hi.assign(K + 1, 0);
  S.A.resize(static_cast<size_t>(K + 1) * dp);
  S.ov_ptr.assign(K + 2, 0);
  std::vector<DD> Ak(dp), gsk(static_cast<size_t>(Jg) * d), gAk(gAf.size());
  std::vector<int64_t> gnk(Jg, 0);
  std::vector<int> touched;
  for (int k = 0; k <= K; ++k) {
    S.ov_ptr[k] = static_cast<int>(S.ov_g.size());
    int t0 = 0, t1 = 0;
    if (k < K && lo[k] < hi[k]) {
      t0 = static_cast<int>(std::lower_bound(skey.begin(), skey.end(), lo[k]) - skey.begin());
      t1 = static_cast<int>(std::lower_bound(skey.begin(), skey.end(), hi[k]) - skey.begin());
    }
    S.ex_lo[k] = t0;
    S.ex_hi[k] = t1;
    std::copy(Af.begin(), Af.end(), Ak.begin());
    std::vector<DD> sk(sf);  // the fold's training sum of u
    touched.clear();
    for (int t = t0; t < t1; ++t) {
      const int r = S.ex_rows[t], g = S.ex_grp[t];
      for (int i = 0; i < d; ++i) {
        dd_add(sk[i], -u(r, i), 0.0);
        for (int j = 0; j <= i; ++j) dd_add_prod(Ak[i * (i + 1) / 2 + j], u(r, i), u(r, j), -1.0);
      }
      if (gnk[g] == 0) {
        touched.push_back(g);
        for (int i = 0; i < d; ++i) gsk[static_cast<size_t>(g) * d + i] = gsf[static_cast<size_t>(g) * d + i];
        if (group_gram)
          for (int e = 0; e < dp; ++e) gAk[static_cast<size_t>(g) * dp + e] = gAf[static_cast<size_t>(g) * dp + e];
      }
      ++gnk[g];
      for (int i = 0; i < d; ++i) dd_add(gsk[static_cast<size_t>(g) * d + i], -u(r, i), 0.0);
      if (group_gram)
        for (int i = 0; i < d; ++i)
          for (int j = 0; j <= i; ++j)
            dd_add_prod(gAk[static_cast<size_t>(g) * dp + i * (i + 1) / 2 + j], u(r, i), u(r, j), -1.0);
    }
    // A' = A - ubar s^T - s ubar^T + n ubar ubar^T (training rows of fold k)
    const double nk = static_cast<double>(n - (t1 - t0));
    for (int i = 0; i < d; ++i)
      for (int j = 0; j <= i; ++j) {
        DD& a = Ak[i * (i + 1) / 2 + j];
        if (ub[i] != 0.0 || ub[j] != 0.0) {
          dd_add_prod(a, ub[i], sk[j].hi, -1.0);
          dd_add(a, -ub[i] * sk[j].lo, 0.0);
          dd_add_prod(a, ub[j], sk[i].hi, -1.0);
          dd_add(a, -ub[j] * sk[i].lo, 0.0);
          const double uu = ub[i] * ub[j], uue = std::fma(ub[i], ub[j], -uu);
          dd_add_prod(a, nk, uu, 1.0);
          dd_add(a, nk * uue, 0.0);
        }
      }
    for (int i = 0; i < dp; ++i) S.A[static_cast<size_t>(k) * dp + i] = dd_val(Ak[i]);
    std::sort(touched.begin(), touched.end());
    for (int g : touched) {
      const int64_t ntr = gnf[g] - gnk[g];
      S.ov_g.push_back(g);
      S.ov_n.push_back(static_cast<double>(ntr));
      for (int i = 0; i < d; ++i)
        S.ov_s.push_back(ntr == 0 ? 0.0 : centred_sum(gsk[static_cast<size_t>(g) * d + i], static_cast<double>(ntr), i));
      if (group_gram)
        for (int e = 0; e < dp; ++e) S.ov_A.push_back(ntr == 0 ? 0.0 : dd_val(gAk[static_cast<size_t>(g) * dp + e]));
      gnk[g] = 0;
    }
  }
  S.ov_ptr[K + 1] = static_cast<int>(S.ov_g.size());
  if (S.ov_g.empty()) {  // keep device pointers valid
    S.ov_g.push_back(-1);
    S.ov_n.push_back(0.0);
    S.ov_s.assign(d, 0.0);
    if (group_gram) S.ov_A.assign(dp, 0.0);
  }
  return true;
}

}  // namespace pcvg
