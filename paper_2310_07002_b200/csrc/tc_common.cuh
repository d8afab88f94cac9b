// sm_100a building blocks of the tensor-core kernels: FP64 DMMA, mbarriers, TMA bulk copies,
// and the cheap FP64 transcendentals the sigmoid needs (DMMA and DFMA share one FP64 datapath on
// B200, measured in tools/probes/fp64_peak.cu, so elementwise FP64 work is taken from the GEMM).
#pragma once
#include <cstdint>

namespace pcvg {
namespace tc {

// D(8x8) += A(8x4, row) * B(4x8, col), FP64 tensor core (SASS DMMA.8x8x4).
// Fragments: lane l holds A[l>>2][l&3], B[l&3][l>>2], D[l>>2][2(l&3) + {0,1}].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)),
               "r"(bytes));
}

// One TMA bulk copy global -> shared completing on `bar` (SASS UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// Address of `p` in the shared memory of cluster rank `rank` (shared::cluster window).
__device__ __forceinline__ uint32_t cluster_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}

// One bulk copy from this CTA's shared memory into another CTA's of the cluster (both addresses
// 16-byte aligned, bytes a multiple of 16), completing on the destination CTA's mbarrier.
__device__ __forceinline__ void bulk_s2c(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "r"(smem_addr(src)), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

// exp(-a) for a >= 0 with ~1 ulp error in 11 FP64 operations (CUDA's exp() spends ~17 plus a
// special-case branch): -a = -(n/16) ln2 + r, |r| <= ln2/32, 2^(-j/16) from a 16-entry table,
// e^r by a degree-6 Taylor polynomial (truncation < 4e-17), 2^(-m) assembled in the exponent.
__device__ __forceinline__ double exp_neg(double a, const double* tab) {
  constexpr double kInvLn2x16 = 23.083120654223414;      // 16 / ln 2
  constexpr double kLn2d16Hi = 0.04332169877307024;      // ln2/16, leading 32 bits
  constexpr double kLn2d16Lo = 1.1926343307941173e-11;   // ln2/16 - hi
  constexpr double kShift = 6755399441055744.0;          // 1.5 * 2^52
  a = fmin(a, 700.0);  // exp(-700) ~ 1e-304 stands in for the underflow; keeps 2^-m in range
  const double t = fma(a, kInvLn2x16, kShift);
  const int n = __double2loint(t);
  const double nd = t - kShift;
  double r = fma(nd, kLn2d16Hi, -a);
  r = fma(nd, kLn2d16Lo, r);
  double p = fma(r, 1.0 / 720.0, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double scale = __hiloint2double((1023 - (n >> 4)) << 20, 0);
  return (tab[n & 15] * scale) * p;
}

// exp(-a) for a >= 0 to ~1.5e-13 relative in 10 FP64 operations: exp_neg with a degree-5
// polynomial (truncation |r|^6/720 <= 1.5e-13 at |r| <= ln2/32). Used where only the logistic
// residual y - sigmoid(eta) needs it: an error d in sigmoid moves a gradient component by at most
// sum_i |x_ij| d, far inside the 1e-12 * sum|terms| parity tolerance.
__device__ __forceinline__ double exp_neg_5(double a, const double* tab) {
  constexpr double kInvLn2x16 = 23.083120654223414;
  constexpr double kLn2d16Hi = 0.04332169877307024;
  constexpr double kLn2d16Lo = 1.1926343307941173e-11;
  constexpr double kShift = 6755399441055744.0;
  a = fmin(a, 700.0);
  const double t = fma(a, kInvLn2x16, kShift);
  const int n = __double2loint(t);
  const double nd = t - kShift;
  double r = fma(nd, kLn2d16Hi, -a);
  r = fma(nd, kLn2d16Lo, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double scale = __hiloint2double((1023 - (n >> 4)) << 20, 0);
  return (tab[n & 15] * scale) * p;
}

// 1 / d for d in [1, 2] to ~1e-13 relative: hardware approximation (~2^-22) + one Newton step.
__device__ __forceinline__ double rcp_1_2_fast(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// y - sigmoid(x) for the gradient-only passes in 11 FP64 operations (exp_neg_5 + rcp_1_2_fast +
// select + subtract cost 18). DMMA and DFMA share one FP64 datapath, so every FP64 operation saved
// here is returned to the GEMM:
// * |x| <= 700 is clamped by an integer compare of the high word (|x| >= 0, so bit order is value
//   order; NaN clamps to 700 exactly as fmin does);
// * -|x| = -(n/32) ln2 + r with ONE reduction constant: ln2/32 is off by 7e-19 in double, so r is
//   off by at most 2.3e-14 (at |x| = 700, where e^-|x| ~ 1e-304) and ~1e-16 where it matters;
// * e^r on |r| <= ln2/64 by a degree-4 Chebyshev-interpolation polynomial (max relative error
//   7.9e-14, tools/exp_poly.py), 2^(-j/32) from a 32-entry table split into high and low words
//   (two 32-word arrays: any 32 indices hit 32 distinct banks, where a double table of 32
//   entries would conflict 2-way);
// * 2^(-j/32) * 2^(-m) subtracts m from the table entry's exponent (exact: the entry is in (0.5, 1]
//   and m <= 1009, so the product stays normal);
// * 1 + e^-|x| is one FMA, and both branches of the sigmoid share the reciprocal:
//   x >= 0: y - 1/(1+e^-|x|);  x < 0: y - e^-|x|/(1+e^-|x|) = (y - 1) + 1/(1+e^-|x|),
//   chosen on the sign bit (x = -0 gives y - 1/2 either way) with ym1 = y - 1 precomputed per row.
//   Both branches carry the reciprocal's absolute error (~1e-14), symmetric in the sign of x.
__device__ __forceinline__ double logistic_resid_fast(double x, double y, double ym1,
                                                      const int* tab_hi, const int* tab_lo) {
  constexpr double kInvLn2x32 = 46.16624130844683;    // 32 / ln 2
  constexpr double kLn2d32 = 0.02166084939249829;     // ln 2 / 32
  constexpr double kShift = 6755399441055744.0;       // 1.5 * 2^52
  constexpr double kC1 = 0.9999999999641696, kC2 = 0.4999999999940276;
  constexpr double kC3 = 0.1666678885252701, kC4 = 0.04166687031843588;
  const int xh = __double2hiint(x);
  const int ah = xh & 0x7fffffff;
  const double a = ah >= 0x4085E000 ? 700.0 : __hiloint2double(ah, __double2loint(x));
  const double t = fma(a, kInvLn2x32, kShift);
  const int n = __double2loint(t);
  const double nd = t - kShift;
  const double r = fma(nd, kLn2d32, -a);
  double p = fma(r, kC4, kC3);
  p = fma(p, r, kC2);
  p = fma(p, r, kC1);
  p = fma(p, r, 1.0);
  const double scaled = __hiloint2double(tab_hi[n & 31] - ((n >> 5) << 20), tab_lo[n & 31]);
  const double inv = rcp_1_2_fast(fma(scaled, p, 1.0));
  const bool pos = xh >= 0;
  return fma(pos ? -1.0 : 1.0, inv, pos ? y : ym1);
}

// 1 / d for d in [1, 2]: hardware approximation + two Newton steps (no special cases needed).
__device__ __forceinline__ double rcp_1_2(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

}  // namespace tc
}  // namespace pcvg
