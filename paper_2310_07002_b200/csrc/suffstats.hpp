// Fold sufficient statistics of the Gaussian linear families (suffstats.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace pcvg {

struct SuffStats {
  int d = 0, dp = 0;                 // d = nc + 1, dp = d (d + 1) / 2
  std::vector<double> A;             // [K+1][dp] packed lower triangle, row i at i (i + 1) / 2
  std::vector<double> gn, gs;        // [Jg], [Jg][d] full-data group counts / sums
  std::vector<int> ov_ptr, ov_g;     // [K+2], [nov]: groups touched by fold k (ascending)
  std::vector<double> ov_n, ov_s;    // [nov], [nov][d]: their training count / sums in fold k
  std::vector<int> ex_lo, ex_hi;     // [K+1]: fold k's excluded rows are ex_rows[ex_lo..ex_hi)
  std::vector<int> ex_rows, ex_grp;  // [n] device rows sorted by key (stable), their group
  std::vector<double> gA, ov_A;      // group_gram: [Jg][dp], [nov][dp] per-group Grams of u
  std::vector<double> ubar;          // [d] centre: A and the group sums are of u - ubar (zeros: uncentred)
};

bool build_suffstats(int64_t n, int nc, int J, const double* y, const double* xc, const int* key,
                     const int* grp_ptr, int K, const int* lo, const int* hi, SuffStats& S,
                     bool group_gram = false, bool center = true);

}  // namespace pcvg
