// Device building blocks shared by the PCV kernels (sm_100a, FP64).
//
//  * ChainRng  - the reference's per-chain CounterRng stream (rng.hpp:45-143) re-expressed as a
//                position-addressable Philox4x32-10 stream: state = (key, stream id, u32 position,
//                cached Box-Muller variate). Integer output is bit-exact with the reference; the
//                Box-Muller transform uses CUDA's FP64 log/sqrt/sincos (<= 1-2 ulp from glibc).
//  * log-space helpers (math.hpp:17-42) and the ScoreAccum update (accum.cpp:101-182).
#pragma once
#include <math_constants.h>

#include <cstdint>

namespace pcvg {

constexpr double kLog2Pi = 1.8378770664093454835606594728112;

// Shuffle-benchmark blocks over stored sub-blocks: with `sub` completed sub-blocks
// regrouped into `groups` blocks, block g covers sub-blocks [begin(g), begin(g + 1)). Without early
// stop sub == groups == RunConfig::blocks and every block is one sub-block (the reference layout,
// accum.cpp:129-156).
__host__ __device__ inline int block_group_begin(int g, int sub, int groups) {
  return static_cast<int>(static_cast<int64_t>(g) * sub / groups);
}
constexpr double kTwoPi = 6.283185307179586476925286766559;

__host__ __device__ inline uint64_t mix64(uint64_t z) {  // rng.hpp:18-23
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t stream_key(uint64_t kind, uint64_t a, uint64_t b,
                                               uint64_t c) {  // rng.hpp:35-43
  uint64_t k = mix64(kind);
  k = mix64(k ^ a);
  k = mix64(k ^ b);
  k = mix64(k ^ c);
  return k;
}

// Philox4x32-10 block `ctr` (64-bit block counter in words 0-1, stream id in words 2-3).
__device__ __forceinline__ uint4 philox_block(uint64_t block, uint64_t stream, uint32_t k0,
                                              uint32_t k1) {
  uint32_t c0 = static_cast<uint32_t>(block), c1 = static_cast<uint32_t>(block >> 32);
  uint32_t c2 = static_cast<uint32_t>(stream), c3 = static_cast<uint32_t>(stream >> 32);
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

// A chain's sequential stream. `pos` counts u32 words consumed since construction, so the
// reference state (ctr, have) maps to pos = 4*ctr - have.
struct ChainRng {
  uint32_t k0, k1;
  uint64_t stream;
  uint64_t pos;
  double cached;
  bool has_cached;
  uint64_t buf_block;  // block held in buf (~0 = none)
  uint4 buf;

  __device__ void init(uint64_t seed, uint64_t stream_id, uint64_t p, double c, bool hc) {
    k0 = static_cast<uint32_t>(seed);
    k1 = static_cast<uint32_t>(seed >> 32);
    stream = stream_id;
    pos = p;
    cached = c;
    has_cached = hc;
    buf_block = ~0ull;
  }
  __device__ __forceinline__ uint32_t next_u32() {  // rng.hpp:58-61
    const uint64_t blk = pos >> 2;
    if (blk != buf_block) {
      buf = philox_block(blk, stream, k0, k1);
      buf_block = blk;
    }
    const uint32_t w = static_cast<uint32_t>(pos & 3);
    ++pos;
    return w == 0 ? buf.x : (w == 1 ? buf.y : (w == 2 ? buf.z : buf.w));
  }
  __device__ __forceinline__ uint64_t next_u64() {  // rng.hpp:63-67
    const uint64_t lo = next_u32();
    const uint64_t hi = next_u32();
    return lo | (hi << 32);
  }
  __device__ __forceinline__ double uniform() {  // rng.hpp:70-72
    return (static_cast<double>(next_u64() >> 11) + 0.5) * 0x1p-53;
  }
  __device__ __forceinline__ double normal() {  // rng.hpp:75-87
    if (has_cached) {
      has_cached = false;
      return cached;
    }
    const double u1 = uniform();
    const double u2 = uniform();
    const double r = sqrt(-2.0 * log(u1));
    double s, c;
    sincos(kTwoPi * u2, &s, &c);
    cached = r * s;
    has_cached = true;
    return r * c;
  }
  __device__ uint64_t below(uint64_t n) {  // rng.hpp:99-105
    const uint64_t bound = n * ((~0ull) / n);
    for (;;) {
      const uint64_t v = next_u64();
      if (v < bound) return v % n;
    }
  }
};

// The Box-Muller pair ChainRng::normal() draws from stream words [wpos, wpos + 4) (two uniforms of
// two words each, rng.hpp:70-87): *a is the value returned first, *b the one cached. Lets several
// threads draw a chain's momenta in parallel at known stream positions with the same bits.
__device__ __forceinline__ void normal_pair_at(uint32_t k0, uint32_t k1, uint64_t stream, uint64_t wpos,
                                               double* a, double* b) {
  const uint64_t blk = wpos >> 2;
  const int o = static_cast<int>(wpos & 3);
  const uint4 x = philox_block(blk, stream, k0, k1);
  uint4 y = x;
  if (o != 0) y = philox_block(blk + 1, stream, k0, k1);
  auto word = [&](int i) -> uint32_t {  // word i (0..7) of blocks blk, blk + 1
    const uint4 v = i < 4 ? x : y;
    const int j = i & 3;
    return j == 0 ? v.x : (j == 1 ? v.y : (j == 2 ? v.z : v.w));
  };
  const uint64_t v1 = static_cast<uint64_t>(word(o)) | (static_cast<uint64_t>(word(o + 1)) << 32);
  const uint64_t v2 = static_cast<uint64_t>(word(o + 2)) | (static_cast<uint64_t>(word(o + 3)) << 32);
  const double u1 = (static_cast<double>(v1 >> 11) + 0.5) * 0x1p-53;
  const double u2 = (static_cast<double>(v2 >> 11) + 0.5) * 0x1p-53;
  const double r = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincos(kTwoPi * u2, &sn, &cs);
  *a = r * cs;
  *b = r * sn;
}

__device__ __forceinline__ double logaddexp(double a, double b) {  // math.hpp:17-22
  if (a == -CUDART_INF) return b;
  if (b == -CUDART_INF) return a;
  const double m = a > b ? a : b;
  return m + log1p(exp(-fabs(a - b)));
}

__device__ __forceinline__ double normal_logpdf(double x, double mean, double var) {
  const double r = x - mean;  // math.hpp:39-42
  return -0.5 * (kLog2Pi + log(var) + r * r / var);
}

// Per-chain online accumulator state, SoA in global memory (accum.hpp:70-127).
struct AccumDev {
  double* u_x;
  double* u_x2;
  double* z_x;
  double* v_x;
  double* v_x2;
  int64_t* committed;
  int32_t* pending;
  int64_t* count;
  int64_t* faults;
  double* center;  // C_k of the chain's fold
  double* y_x;     // [D][nch]
  double* y_x2;    // [D][nch]
};

// ScoreAccum::observe (accum.cpp:164-182) for chain c at sampling iteration iter.
__device__ inline void accum_observe(const AccumDev& A, int c, int nch, double s, int64_t iter,
                                     int64_t planned_n, int D, int b) {
  int64_t blk = planned_n <= 0 ? 0 : iter * D / planned_n;  // accum.cpp:134-139
  if (blk >= D) blk = D - 1;
  double centred;
  if (isnan(s) || (isinf(s) && s > 0.0)) {
    A.faults[c] += 1;
    s = -CUDART_INF;
    centred = 0.0;
  } else {
    centred = s - A.center[c];
  }
  A.u_x[c] = logaddexp(A.u_x[c], s);
  A.u_x2[c] = logaddexp(A.u_x2[c], 2.0 * s);
  double z = logaddexp(A.z_x[c], s);  // BatchState::add, accum.cpp:115-127
  int32_t pend = A.pending[c] + 1;
  if (pend == b) {
    const double log_mean = z - log(static_cast<double>(b));
    A.v_x[c] = logaddexp(A.v_x[c], log_mean);
    A.v_x2[c] = logaddexp(A.v_x2[c], 2.0 * log_mean);
    z = -CUDART_INF;
    pend = 0;
    A.committed[c] += 1;
  }
  A.z_x[c] = z;
  A.pending[c] = pend;
  A.y_x[blk * nch + c] += centred;
  A.y_x2[blk * nch + c] += centred * centred;
  A.count[c] += 1;
}

}  // namespace pcvg
