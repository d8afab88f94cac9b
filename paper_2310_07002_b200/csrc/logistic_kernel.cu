// Fused HMC kernel for the Bernoulli-logit family (BASELINE configs[1]: N=10k, P=50, 10k LOO
// folds x 8 chains) on sm_100a, FP64.
//
// The per-chain gradient sum_i [y_i - sigmoid(x_i . theta)] x_i over N observations is
// GEMM-shaped across the 64 chains of a CTA:  eta = X_tile . Theta  ->  R = mask(y - sigmoid(eta))
// ->  G += X_tile^T . R. Both contractions run on the FP64 tensor cores (DMMA,
// mma.sync.m8n8k4.f64: 37 TF/s measured on B200; DMMA and DFMA share one FP64 datapath, so the
// sigmoid is written to spend as few FP64 operations as possible). The N x chains predictor is
// never materialised beyond one 64-row tile. X row tiles (augmented with the intercept column,
// [N][52] row-major, L2-resident: 4.2 MB) stream into a 3-stage shared-memory ring by TMA bulk
// copies (cp.async.bulk + full/empty mbarriers) issued by one thread. 16 warps = 4 row quarters x
// 4 chain groups; each warp reads back only its own R block, so the phases of different warps
// drift freely within the ring and overlap. Chain positions live in shared memory (the tensor-core
// B operand); momenta in the registers of 8 owner threads per chain; RNG / energies / accept /
// log_pred / accumulators in one "chain thread" per chain. Semantics follow hmc.cpp:22-99 and
// engine.cpp:342-381 (see gauss_kernel.cu for the shared conventions).
#include <math_constants.h>

#include "device_common.cuh"
#include "types.cuh"

namespace pcvg {

namespace {

constexpr int kC = 64;          // chains per CTA
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kTM = 64;         // rows per tile
constexpr int kKP = 52;         // padded parameter count (intercept + P <= 51 covariates + pad)
constexpr int kLdS = 68;        // leading dim of [k][chain] / [row][chain] shared arrays
constexpr int kOwners = kThreads / kC;               // owner threads per chain (8)
constexpr int kOwn = (kKP + kOwners - 1) / kOwners;  // dims per owner thread (7)
constexpr int kStages = 3;      // TMA ring depth
constexpr int kTileBytes = kTM * kKP * 8 + kTM * 8 + kTM * 4;

struct Smem {
  double xs[kStages][kTM * kKP + 8];  // +8: the 7th p-tile of X^T overreads 4 doubles past row 63
  double ys[kStages][kTM];
  int ks[kStages][kTM];
  double rs[kTM * kLdS];        // per-warp R blocks; reused as G [kKP][kLdS] and momentum staging
  double qs[kKP * kLdS];        // working positions, [k][chain]
  double llp[4][kC];            // log-likelihood partial per row quarter
  double red[kOwners][kC];      // owner partial sums (kinetic)
  double pri[kOwners][kC];      // owner partial sums (prior)
  double exp_tab[16];           // 2^(-j/16)
  int lo[kC], hi[kC];
  int bad[kC];
  int cur[kC];
  unsigned long long full[kStages];   // tile landed (TMA transaction count)
  unsigned long long empty[kStages];  // all warps done with the slot
};

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

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)),
               "r"(bytes));
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
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

// Producer side of the ring (thread 0): global tile sequence number g (continuing across passes)
// goes to slot g % kStages; before re-filling a slot wait until its previous occupant (g - kStages)
// was released by all warps.
__device__ __forceinline__ void issue_tile(Smem& sm, const ModelDev& M, int t, uint32_t g) {
  const int slot = g % kStages;
  if (g >= kStages) mbar_wait(&sm.empty[slot], ((g - kStages) / kStages) & 1u);
  mbar_expect_tx(&sm.full[slot], kTileBytes);
  bulk_g2s(sm.xs[slot], M.xr + static_cast<size_t>(t) * kTM * kKP, kTM * kKP * 8, &sm.full[slot]);
  bulk_g2s(sm.ys[slot], M.y + static_cast<size_t>(t) * kTM, kTM * 8, &sm.full[slot]);
  bulk_g2s(sm.ks[slot], M.key + static_cast<size_t>(t) * kTM, kTM * 4, &sm.full[slot]);
}

// exp(-a) for a >= 0 with ~1 ulp error in 11 FP64 operations (CUDA's exp() spends ~17 and a
// special-case branch): -a = -(n/16) ln2 + r, |r| <= ln2/32, 2^(-j/16) from a 16-entry table,
// e^r by a degree-6 Taylor polynomial (truncation < 4e-17), 2^(-m) assembled in the exponent.
__device__ __forceinline__ double exp_neg(double a, const double* tab) {
  constexpr double kInvLn2x16 = 23.083120654223414;      // 16 / ln 2
  constexpr double kLn2d16Hi = 0.04332169877307024;      // ln2/16, leading 32 bits
  constexpr double kLn2d16Lo = 1.1926343307941173e-11;   // ln2/16 - hi
  constexpr double kShift = 6755399441055744.0;          // 1.5 * 2^52
  if (a > 700.0) return 0.0;
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

// 1 / d for d in [1, 2]: hardware approximation + two Newton steps (no special cases needed).
__device__ __forceinline__ double rcp_1_2(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// One pass over all observations for the 64 chains at positions sm.qs: G = X^T (y - sigmoid(X q))
// over training rows into sm.rs as [k][chain]; with VALUE, the masked Bernoulli log-likelihood per
// chain into sm.llp[*][c] (NaN-poisoned like the reference's 0 * non-finite test term).
template <bool VALUE>
__device__ void grad_pass(Smem& sm, const ModelDev& M, uint32_t& gtile) {
  const int tid = threadIdx.x;
  const int w = tid >> 5, l = tid & 31;
  const int cg = w & 3, rq = w >> 2;   // chain group (16 chains), row quarter (16 rows)
  const int ntiles = (M.n + kTM - 1) / kTM;
  const uint32_t g0 = gtile;
  if (tid == 0)
    for (int t = 0; t < kStages && t < ntiles; ++t) issue_tile(sm, M, t, g0 + t);
  int lo[2][2], hi[2][2];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int ch = 16 * cg + 8 * j + 2 * (l & 3) + e;
      lo[j][e] = sm.lo[ch];
      hi[j][e] = sm.hi[ch];
    }
  const double* qcol = sm.qs + 16 * cg + (l >> 2);  // B fragments: qs[4ks + (l&3)][16cg + 8j + (l>>2)]
  double gacc[7][2][2];
#pragma unroll
  for (int pt = 0; pt < 7; ++pt)
#pragma unroll
    for (int j = 0; j < 2; ++j) gacc[pt][j][0] = gacc[pt][j][1] = 0.0;
  double ll[2][2] = {{0.0, 0.0}, {0.0, 0.0}};

  for (int t = 0; t < ntiles; ++t) {
    const uint32_t g = g0 + t;
    const int slot = g % kStages;
    mbar_wait(&sm.full[slot], (g / kStages) & 1u);
    const double* xs = sm.xs[slot];
    // eta = X_tile . Q   (rows 16rq .. 16rq+15, chains 16cg .. 16cg+15)
    double eta[2][2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int j = 0; j < 2; ++j) eta[mt][j][0] = eta[mt][j][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 13; ++ks) {
      double b[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = qcol[(4 * ks + (l & 3)) * kLdS + 8 * j];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const double a = xs[(16 * rq + 8 * mt + (l >> 2)) * kKP + 4 * ks + (l & 3)];
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(eta[mt][j][0], eta[mt][j][1], a, b[j]);
      }
    }
    // R = train ? y - sigmoid(eta) : 0 into this warp's private 16 x 16 block of sm.rs
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int row = 16 * rq + 8 * mt + (l >> 2);
      const bool valid = t * kTM + row < M.n;
      const double yv = sm.ys[slot][row];
      const int kv = sm.ks[slot][row];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double r2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double x = eta[mt][j][e];
          const bool train =
              valid && static_cast<unsigned>(kv - lo[j][e]) >= static_cast<unsigned>(hi[j][e] - lo[j][e]);
          const double ex = exp_neg(fabs(x), sm.exp_tab);
          const double inv = rcp_1_2(1.0 + ex);
          const double sig = x >= 0.0 ? inv : ex * inv;
          r2[e] = train ? yv - sig : 0.0;
          if (VALUE) {
            if (train) ll[j][e] += yv * x - (fmax(x, 0.0) + log1p(ex));
            else if (valid && !isfinite(x)) ll[j][e] = CUDART_NAN;  // 0 * non-finite test term
          }
        }
        *reinterpret_cast<double2*>(&sm.rs[row * kLdS + 16 * cg + 8 * j + 2 * (l & 3)]) =
            make_double2(r2[0], r2[1]);
      }
    }
    __syncwarp();
    // G += X_tile^T . R   (k rows 16rq .. 16rq+15; this warp's own R block)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int m = 16 * rq + 4 * ks + (l & 3);
      double b[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = sm.rs[m * kLdS + 16 * cg + 8 * j + (l >> 2)];
#pragma unroll
      for (int pt = 0; pt < 7; ++pt) {
        const double a = xs[m * kKP + 8 * pt + (l >> 2)];
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(gacc[pt][j][0], gacc[pt][j][1], a, b[j]);
      }
    }
    __syncwarp();
    if (l == 0) mbar_arrive(&sm.empty[slot]);
    if (tid == 0 && t + kStages < ntiles) issue_tile(sm, M, t + kStages, g + kStages);
  }
  gtile = g0 + ntiles;
  __syncthreads();  // every warp is done with every tile and with its R block
  // Stage G [k][chain] into sm.rs: row quarter 0 stores, quarters 1..3 add in order.
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    if (rq == q) {
#pragma unroll
      for (int pt = 0; pt < 7; ++pt) {
        const int p = 8 * pt + (l >> 2);
        if (p < kKP) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            double2* dst = reinterpret_cast<double2*>(&sm.rs[p * kLdS + 16 * cg + 8 * j + 2 * (l & 3)]);
            if (q == 0) {
              *dst = make_double2(gacc[pt][j][0], gacc[pt][j][1]);
            } else {
              const double2 v = *dst;
              *dst = make_double2(v.x + gacc[pt][j][0], v.y + gacc[pt][j][1]);
            }
          }
        }
      }
      if (VALUE) {
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double v = ll[j][e];
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            if (l < 4) sm.llp[q][16 * cg + 8 * j + 2 * l + e] = v;
          }
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double bernoulli_logit(double y, double x) {
  return y * x - (fmax(x, 0.0) + log1p(exp(-fabs(x))));
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1) logistic_kernel(ModelDev M, ChainsDev S, RunArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int nch = S.nch;
  const int dim = M.dim;
  const size_t plane = static_cast<size_t>(dim) * nch;
  // owner role: chain oc, dims k = ok + kOwners*j
  const int oc = tid & (kC - 1), ok = tid / kC;
  const int ogc = blockIdx.x * kC + oc;
  const bool ovalid = ogc < nch;
  // chain-thread role
  const bool is_chain = tid < kC;
  const int gc = blockIdx.x * kC + tid;
  const bool cvalid = is_chain && gc < nch;

  if (tid < kStages) {
    mbar_init(&sm.full[tid], 1);
    mbar_init(&sm.empty[tid], kWarps);
  }
  if (tid < 16) sm.exp_tab[tid] = exp2(-tid / 16.0);
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
      sm.cur[tid] = S.cur[gc];
      lp0 = S.lp0[gc];
      R.init(S.seed, S.rng_stream[gc], S.rng_pos[gc], S.rng_cached[gc], S.rng_has[gc] != 0);
    } else {
      sm.lo[tid] = 0;
      sm.hi[tid] = 0;
      sm.cur[tid] = 0;
    }
  }
  __syncthreads();

  auto lp_from_partials = [&](int c) {
    double pr = 0.0;
#pragma unroll
    for (int o = 0; o < kOwners; ++o) pr += sm.pri[o][c];
    return ((sm.llp[0][c] + sm.llp[1][c]) + (sm.llp[2][c] + sm.llp[3][c])) + pr;
  };

  if (A.mode == kModeEval) {
    {
      const int cu = sm.cur[oc];
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        const int k = ok + kOwners * j;
        if (k < kKP)
          sm.qs[k * kLdS + oc] = (ovalid && k < dim) ? S.pos[cu * plane + static_cast<size_t>(k) * nch + ogc] : 0.0;
      }
    }
    __syncthreads();
    grad_pass<true>(sm, M, gtile);
    // gradient = likelihood part - theta (beta_j ~ N(0,1)); prior partials of the log joint
    double pr = 0.0;
    const int cu = sm.cur[oc];
#pragma unroll
    for (int j = 0; j < kOwn; ++j) {
      const int k = ok + kOwners * j;
      if (k < dim) {
        const double q = sm.qs[k * kLdS + oc];
        if (ovalid) S.grad[cu * plane + static_cast<size_t>(k) * nch + ogc] = sm.rs[k * kLdS + oc] - q;
        pr += -0.5 * (kLog2Pi + q * q);
      }
    }
    sm.pri[ok][oc] = pr;
    __syncthreads();
    if (cvalid) {
      const double lp = lp_from_partials(tid);
      S.lp0[gc] = lp;
      if (A.out_a) A.out_a[gc] = lp;
    }
    return;
  }

  const double eps = M.step, half = 0.5 * M.step;
  const int n_lf = M.n_lf;
  for (int64_t it = 0; it < A.n_iters; ++it) {
    if (A.mode != kModePred) {
      // -- momentum refresh (chain thread, reference draw order) -> staging in sm.rs
      double k0 = 0.0;
      if (is_chain) {
        for (int k = 0; k < kKP; ++k) {
          double p = 0.0;
          if (k < dim) {
            const double mk = __ldg(M.inv_mass + k);
            if (A.mode == kModeProbe) p = cvalid ? A.probe_momentum[static_cast<size_t>(gc) * dim + k] : 0.0;
            else p = R.normal() / sqrt(mk);
            k0 += mk * p * p;
          }
          sm.rs[k * kLdS + tid] = p;
        }
        sm.bad[tid] = 0;
      }
      __syncthreads();
      // -- half kick + first drift (owners)
      double pown[kOwn];
      {
        const int cu = sm.cur[oc];
        bool bad = false;
#pragma unroll
        for (int j = 0; j < kOwn; ++j) {
          const int k = ok + kOwners * j;
          double q = 0.0, p = 0.0;
          if (k < dim && ovalid) {
            const size_t gi = cu * plane + static_cast<size_t>(k) * nch + ogc;
            p = sm.rs[k * kLdS + oc] + half * S.grad[gi];
            q = S.pos[gi] + eps * __ldg(M.inv_mass + k) * p;
            bad |= !isfinite(q);
          }
          pown[j] = p;
          if (k < kKP) sm.qs[k * kLdS + oc] = q;
        }
        if (bad) sm.bad[oc] = 1;
      }
      __syncthreads();
      // -- leapfrog: n_lf gradient passes
      for (int s = 0; s < n_lf; ++s) {
        const bool last = s == n_lf - 1;
        if (last) grad_pass<true>(sm, M, gtile);
        else grad_pass<false>(sm, M, gtile);
        const double scale = last ? half : eps;
        const int cu = sm.cur[oc];
        bool bad = false;
        double part = 0.0, part2 = 0.0;
#pragma unroll
        for (int j = 0; j < kOwn; ++j) {
          const int k = ok + kOwners * j;
          if (k < dim) {
            const double q = sm.qs[k * kLdS + oc];
            const double g = sm.rs[k * kLdS + oc] - q;
            bad |= !isfinite(g);
            pown[j] += scale * g;
            bad |= !isfinite(pown[j]);
            if (last) {
              const double mk = __ldg(M.inv_mass + k);
              part += mk * pown[j] * pown[j];
              part2 += -0.5 * (kLog2Pi + q * q);
              if (ovalid) {
                const size_t gi = (cu ^ 1) * plane + static_cast<size_t>(k) * nch + ogc;
                S.pos[gi] = q;
                S.grad[gi] = g;
              }
            }
          }
        }
        __syncthreads();  // all owners read G/q before they are overwritten
        if (!last) {
#pragma unroll
          for (int j = 0; j < kOwn; ++j) {
            const int k = ok + kOwners * j;
            if (k < dim) {
              const double q = sm.qs[k * kLdS + oc] + eps * __ldg(M.inv_mass + k) * pown[j];
              bad |= !isfinite(q);
              sm.qs[k * kLdS + oc] = q;
            }
          }
        } else {
          sm.red[ok][oc] = part;
          sm.pri[ok][oc] = part2;
        }
        if (bad) sm.bad[oc] = 1;
        __syncthreads();
      }
      // -- energies, Metropolis (chain thread)
      if (is_chain) {
        double k1 = 0.0;
#pragma unroll
        for (int o = 0; o < kOwners; ++o) k1 += sm.red[o][tid];
        const double lp1 = lp_from_partials(tid);
        const bool bad = sm.bad[tid] != 0;
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
        if (cvalid && A.mode == kModeProbe) {
          A.out_a[gc] = h0;
          A.out_b[gc] = h1;
          A.out_flags[gc] = (accepted ? 1 : 0) | (divergent ? 2 : 0);
        }
        if (cvalid && A.mode == kModeChain) A.traj_div[it] = divergent ? 1 : 0;
      }
      __syncthreads();
      if (A.mode == kModeProbe) continue;
      if (A.mode == kModeChain) {
        const int cu = sm.cur[oc];
        if (ovalid) {
#pragma unroll
          for (int j = 0; j < kOwn; ++j) {
            const int k = ok + kOwners * j;
            if (k < dim) A.traj[it * dim + k] = S.pos[cu * plane + static_cast<size_t>(k) * nch + ogc];
          }
        }
        continue;
      }
    }
    // -- log_pred at the current position + accumulators (chain thread)
    if (cvalid) {
      double sp = 0.0;
      if (fold < M.K) {
        const int cu = sm.cur[tid];
        const int s0 = M.fold_seg[fold], s1 = M.fold_seg[fold + 1];
        for (int s = s0; s < s1; ++s) {
          for (int tt = M.seg_row[s]; tt < M.seg_row[s + 1]; ++tt) {
            const int i = M.seg_rows[tt];
            const double* xrow = M.xr + static_cast<size_t>(i) * M.nc_pad;
            double eta = 0.0;
            for (int k = 0; k < dim; ++k) eta = fma(xrow[k], S.pos[cu * plane + static_cast<size_t>(k) * nch + gc], eta);
            sp += bernoulli_logit(M.y[i], eta);
          }
        }
      }
      if (A.mode == kModePred) {
        if (A.out_a) A.out_a[gc] = sp;
      } else if (A.mode == kModeWarmup) {
        warm += sp;
      } else {
        accum_observe(S.acc, gc, nch, sp, A.iter0 + it, A.planned_n, A.D, A.b);
      }
    }
    if (A.mode == kModePred) break;
  }
  if (cvalid && A.mode != kModePred) {
    S.cur[gc] = static_cast<int8_t>(sm.cur[tid]);
    S.lp0[gc] = lp0;
    S.rng_pos[gc] = R.pos;
    S.rng_cached[gc] = R.cached;
    S.rng_has[gc] = R.has_cached ? 1 : 0;
    S.divergences[gc] += div_count;
    if (A.mode == kModeWarmup) S.warm_sum[gc] += warm;
  }
}

size_t logistic_smem_bytes() { return sizeof(Smem); }

cudaError_t launch_logistic(const ModelDev& M, const ChainsDev& S, const RunArgs& A,
                            cudaStream_t st) {
  if (M.nc_pad != kKP || M.dim > kKP) return cudaErrorInvalidValue;
  const int grid = (S.nch + kC - 1) / kC;
  if (grid == 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(logistic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sizeof(Smem)));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  logistic_kernel<<<grid, kThreads, sizeof(Smem), st>>>(M, S, A);
  return cudaGetLastError();
}

}  // namespace pcvg
