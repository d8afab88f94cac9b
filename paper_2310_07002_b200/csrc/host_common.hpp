// Host-side restatements that must be bit-exact with the reference: the Philox CounterRng
// (rng.hpp:45-143), fold schemes (folds.cpp:43-108) and the data simulators. Pure C++.
#pragma once
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "device_common.cuh"

namespace pcvg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// CounterRng, rng.hpp:45-143.
class HostRng {
 public:
  HostRng(uint64_t seed, uint64_t stream) {
    key_[0] = static_cast<uint32_t>(seed);
    key_[1] = static_cast<uint32_t>(seed >> 32);
    ctr_[0] = ctr_[1] = 0;
    ctr_[2] = static_cast<uint32_t>(stream);
    ctr_[3] = static_cast<uint32_t>(stream >> 32);
  }
  uint32_t next_u32() {
    if (have_ == 0) refill();
    return buf_[4 - have_--];
  }
  uint64_t next_u64() {
    const uint64_t lo = next_u32();
    const uint64_t hi = next_u32();
    return lo | (hi << 32);
  }
  double uniform() { return (static_cast<double>(next_u64() >> 11) + 0.5) * 0x1p-53; }
  double normal() {
    if (has_cached_) {
      has_cached_ = false;
      return cached_;
    }
    const double u1 = uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    cached_ = r * std::sin(a);
    has_cached_ = true;
    return r * std::cos(a);
  }
  void skip_to(uint64_t block) {
    ctr_[0] = static_cast<uint32_t>(block);
    ctr_[1] = static_cast<uint32_t>(block >> 32);
    have_ = 0;
    has_cached_ = false;
  }
  // Device stream state (device_common.cuh ChainRng): u32 words consumed, Box-Muller cache.
  uint64_t position() const {
    return 4 * ((static_cast<uint64_t>(ctr_[1]) << 32) | ctr_[0]) - static_cast<uint64_t>(have_);
  }
  double cached() const { return cached_; }
  bool has_cached() const { return has_cached_; }
  uint64_t below(uint64_t n) {
    const uint64_t bound = n * ((~uint64_t{0}) / n);
    for (;;) {
      const uint64_t v = next_u64();
      if (v < bound) return v % n;
    }
  }

 private:
  void refill() {
    uint32_t c0 = ctr_[0], c1 = ctr_[1], c2 = ctr_[2], c3 = ctr_[3];
    uint32_t k0 = key_[0], k1 = key_[1];
    for (int round = 0; round < 10; ++round) {
      const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
      const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
      c0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ k0;
      c1 = static_cast<uint32_t>(p1);
      c2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ k1;
      c3 = static_cast<uint32_t>(p0);
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    buf_[0] = c0;
    buf_[1] = c1;
    buf_[2] = c2;
    buf_[3] = c3;
    have_ = 4;
    if (++ctr_[0] == 0) ++ctr_[1];
  }
  uint32_t key_[2];
  uint32_t ctr_[4];
  uint32_t buf_[4] = {0, 0, 0, 0};
  int have_ = 0;
  double cached_ = 0.0;
  bool has_cached_ = false;
};

// Marsaglia-Tsang Gamma(a, rate r) (priors.hpp:29-48).
inline double gamma_draw(HostRng& rng, double a, double r) {
  double boost = 1.0;
  if (a < 1.0) {
    boost = std::pow(rng.uniform(), 1.0 / a);
    a += 1.0;
  }
  const double d = a - 1.0 / 3.0;
  const double c = 1.0 / std::sqrt(9.0 * d);
  for (;;) {
    double x, v;
    do {
      x = rng.normal();
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    const double u = rng.uniform();
    if (std::log(u) < 0.5 * x * x + d - d * v + d * std::log(v)) return boost * d * v / r;
  }
}

// beta_draw (priors.hpp:50-54).
inline double beta_draw(HostRng& rng, double a, double b) {
  const double x = gamma_draw(rng, a, 1.0);
  const double y = gamma_draw(rng, b, 1.0);
  return x / (x + y);
}

// Ground truth of a simulated dataset (the `<family>_truth.json` sidecar, registry.cpp:99-160):
// vectors and scalars by name.
struct SimTruth {
  std::vector<std::pair<std::string, std::vector<double>>> vectors;
  std::vector<std::pair<std::string, double>> scalars;
};

// Host simulators (host_folds.cpp); `truth` may be null.
void simulate_grouped(int32_t J, int32_t Nj, int32_t P, double min_beta, uint64_t seed, double* y,
                      double* x, int32_t* g, SimTruth* truth = nullptr);
void simulate_rat(int32_t subjects, uint64_t seed, double* y, double* x, int32_t* g,
                  SimTruth* truth = nullptr);
void simulate_radon(int32_t houses, int32_t counties, uint64_t seed, double* y, double* x,
                    int32_t* g, SimTruth* truth = nullptr);
void simulate_seasonal(int64_t months, int32_t p, int32_t q, double rho, double amp, double sigma,
                       uint64_t seed, double* y, double* x, int64_t* t, SimTruth* truth = nullptr);

// Stable argsort by time (std::stable_sort in folds.cpp:95-98).
std::vector<int64_t> time_order(const int64_t* t, int64_t n);

}  // namespace pcvg
