// Fused HMC kernel for the Bernoulli-logit family (BASELINE configs[1]: N=10k, P=50, 10k LOO
// folds x 8 chains) on sm_100a, FP64.
//
// The per-chain gradient sum_i [y_i - sigmoid(x_i . theta)] x_i over N observations is
// GEMM-shaped across the 64 chains of a CTA:  eta = X_tile . Theta  ->  R = mask(y - sigmoid(eta))
// ->  G += X_tile^T . R. Both contractions run on the FP64 tensor cores (DMMA,
// mma.sync.m8n8k4.f64; measured 37.2 TF/s vs 34.2 TF/s for DFMA on B200); the N x chains predictor
// is never materialised beyond one 64-row tile. X row tiles (augmented with the intercept column,
// [N][52] row-major, L2-resident: 4.2 MB) stream into a double-buffered shared-memory ring by TMA
// bulk copies (cp.async.bulk + mbarrier) issued by one thread, overlapping the DMMA work of the
// previous tile. Chain positions live in shared memory for the tensor-core B operand; momenta in
// the registers of 4 owner threads per chain; RNG / energies / accept / log_pred / accumulators in
// one "chain thread" per chain. Semantics follow hmc.cpp:22-99 and engine.cpp:342-381 (see
// gauss_kernel.cu for the shared conventions).
#include <math_constants.h>

#include "device_common.cuh"
#include "types.cuh"

namespace pcvg {

namespace {

constexpr int kC = 64;       // chains per CTA
constexpr int kThreads = 256;
constexpr int kTM = 64;      // rows per tile
constexpr int kKP = 52;      // padded parameter count (intercept + P <= 51 covariates + pad)
constexpr int kLdS = 68;     // leading dim of [k][chain] shared arrays (bank-conflict padding)
constexpr int kOwn = kKP / 4;  // dims owned per owner thread (13)
constexpr int kTileBytes = kTM * kKP * 8 + kTM * 8 + kTM * 4;

struct Smem {
  double xs[2][kTM * kKP + 8];  // +8: the 7th p-tile of X^T overreads 4 doubles past row 63
  double ys[2][kTM];
  int ks[2][kTM];
  double rs[kTM * kLdS];        // R tile; reused as G [kKP][kLdS] and momentum staging
  double qs[kKP * kLdS];        // working positions, [k][chain]
  double llp[2][kC];            // log-lik partial per row-half
  double red[4][kC];            // owner partial sums (kinetic / prior)
  int lo[kC], hi[kC];
  int bad[kC];
  int cur[kC];
  int accept[kC];
  unsigned long long mbar[2];
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(bar)));
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

// Issues the three bulk copies of row tile `t` into ring slot `buf`.
__device__ __forceinline__ void issue_tile(Smem& sm, const ModelDev& M, int t, int buf) {
  mbar_expect_tx(&sm.mbar[buf], kTileBytes);
  bulk_g2s(sm.xs[buf], M.xr + static_cast<size_t>(t) * kTM * kKP, kTM * kKP * 8, &sm.mbar[buf]);
  bulk_g2s(sm.ys[buf], M.y + static_cast<size_t>(t) * kTM, kTM * 8, &sm.mbar[buf]);
  bulk_g2s(sm.ks[buf], M.key + static_cast<size_t>(t) * kTM, kTM * 4, &sm.mbar[buf]);
}

// One pass over all observations for the 64 chains at positions sm.qs: G = X^T (y - sigmoid(X q))
// over training rows into sm.rs as [k][chain]; with VALUE, the masked Bernoulli log-likelihood per
// chain into sm.llp[0][c] (NaN-poisoned like the reference's 0 * non-finite test term).
template <bool VALUE>
__device__ void grad_pass(Smem& sm, const ModelDev& M, uint32_t (&phase)[2]) {
  const int tid = threadIdx.x;
  const int w = tid >> 5, l = tid & 31;
  const int cg = w & 3, h = w >> 2;
  const int ntiles = (M.n + kTM - 1) / kTM;
  if (tid == 0) {
    issue_tile(sm, M, 0, 0);
    if (ntiles > 1) issue_tile(sm, M, 1, 1);
  }
  double qf[13][2];
#pragma unroll
  for (int ks = 0; ks < 13; ++ks)
#pragma unroll
    for (int j = 0; j < 2; ++j) qf[ks][j] = sm.qs[(4 * ks + (l & 3)) * kLdS + 16 * cg + 8 * j + (l >> 2)];
  int lo[2][2], hi[2][2];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int ch = 16 * cg + 8 * j + 2 * (l & 3) + e;
      lo[j][e] = sm.lo[ch];
      hi[j][e] = sm.hi[ch];
    }
  double gacc[7][2][2];
#pragma unroll
  for (int pt = 0; pt < 7; ++pt)
#pragma unroll
    for (int j = 0; j < 2; ++j) gacc[pt][j][0] = gacc[pt][j][1] = 0.0;
  double ll[2][2] = {{0.0, 0.0}, {0.0, 0.0}};

  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    mbar_wait(&sm.mbar[buf], phase[buf]);
    phase[buf] ^= 1u;
    const double* xs = sm.xs[buf];
    // eta = X_tile . Q   (rows 32h .. 32h+31, chains 16cg .. 16cg+15)
    double eta[4][2][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int j = 0; j < 2; ++j) eta[mt][j][0] = eta[mt][j][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 13; ++ks) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const double a = xs[(32 * h + 8 * mt + (l >> 2)) * kKP + 4 * ks + (l & 3)];
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(eta[mt][j][0], eta[mt][j][1], a, qf[ks][j]);
      }
    }
    // R = train ? y - sigmoid(eta) : 0
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int row = 32 * h + 8 * mt + (l >> 2);
      const bool valid = t * kTM + row < M.n;
      const double yv = sm.ys[buf][row];
      const int kv = sm.ks[buf][row];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double x = eta[mt][j][e];
          const bool train =
              valid && static_cast<unsigned>(kv - lo[j][e]) >= static_cast<unsigned>(hi[j][e] - lo[j][e]);
          const double ex = exp(-fabs(x));
          const double inv = 1.0 / (1.0 + ex);
          const double sig = x >= 0.0 ? inv : ex * inv;
          sm.rs[row * kLdS + 16 * cg + 8 * j + 2 * (l & 3) + e] = train ? yv - sig : 0.0;
          if (VALUE) {
            if (train) ll[j][e] += yv * x - (fmax(x, 0.0) + log1p(ex));
            else if (valid && !isfinite(x)) ll[j][e] = CUDART_NAN;  // 0 * non-finite test term
          }
        }
    }
    __syncthreads();
    // G += X_tile^T . R   (k rows 32h .. 32h+31)
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int m = 32 * h + 4 * ks + (l & 3);
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
    __syncthreads();
    if (tid == 0 && t + 2 < ntiles) issue_tile(sm, M, t + 2, buf);
  }
  // Stage G [k][chain] into sm.rs: row half 0 stores, row half 1 adds.
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    if (h == half) {
#pragma unroll
      for (int pt = 0; pt < 7; ++pt) {
        const int p = 8 * pt + (l >> 2);
        if (p < kKP) {
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              double& dst = sm.rs[p * kLdS + 16 * cg + 8 * j + 2 * (l & 3) + e];
              dst = half == 0 ? gacc[pt][j][e] : dst + gacc[pt][j][e];
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
            if (l < 4) sm.llp[half][16 * cg + 8 * j + 2 * l + e] = v;
          }
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double sigmoid_ll(double y, double x) {
  const double ex = exp(-fabs(x));
  return y * x - (fmax(x, 0.0) + log1p(ex));
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1) logistic_kernel(ModelDev M, ChainsDev S, RunArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int nch = S.nch;
  const int dim = M.dim;
  const size_t plane = static_cast<size_t>(dim) * nch;
  // owner role: chain oc, dims k = ok + 4j
  const int oc = tid & (kC - 1), ok = tid >> 6;
  const int ogc = blockIdx.x * kC + oc;
  const bool ovalid = ogc < nch;
  // chain-thread role
  const bool is_chain = tid < kC;
  const int gc = blockIdx.x * kC + tid;
  const bool cvalid = is_chain && gc < nch;

  if (tid < 2) mbar_init(&sm.mbar[tid]);
  fence_mbar_init();
  uint32_t phase[2] = {0u, 0u};

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

  // Load current positions into sm.qs.
  auto load_q = [&](void) {
    const int cu = sm.cur[oc];
#pragma unroll
    for (int j = 0; j < kOwn; ++j) {
      const int k = ok + 4 * j;
      sm.qs[k * kLdS + oc] = (ovalid && k < dim) ? S.pos[cu * plane + static_cast<size_t>(k) * nch + ogc] : 0.0;
    }
  };

  if (A.mode == kModeEval) {
    load_q();
    __syncthreads();
    grad_pass<true>(sm, M, phase);
    // gradient = likelihood part - theta (beta_j ~ N(0,1)); prior partials of the log joint
    double pr = 0.0;
    const int cu = sm.cur[oc];
#pragma unroll
    for (int j = 0; j < kOwn; ++j) {
      const int k = ok + 4 * j;
      if (k < dim) {
        const double q = sm.qs[k * kLdS + oc];
        if (ovalid) S.grad[cu * plane + static_cast<size_t>(k) * nch + ogc] = sm.rs[k * kLdS + oc] - q;
        pr += -0.5 * (kLog2Pi + q * q);
      }
    }
    sm.red[ok][oc] = pr;
    __syncthreads();
    if (cvalid) {
      const double lp = sm.llp[0][tid] + sm.llp[1][tid] + (sm.red[0][tid] + sm.red[1][tid] + sm.red[2][tid] + sm.red[3][tid]);
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
          const int k = ok + 4 * j;
          double q = 0.0, p = 0.0;
          if (k < dim && ovalid) {
            const size_t gi = cu * plane + static_cast<size_t>(k) * nch + ogc;
            p = sm.rs[k * kLdS + oc] + half * S.grad[gi];
            q = S.pos[gi] + eps * __ldg(M.inv_mass + k) * p;
            bad |= !isfinite(q);
          }
          pown[j] = p;
          sm.qs[k * kLdS + oc] = q;
        }
        if (bad) sm.bad[oc] = 1;
      }
      __syncthreads();
      // -- leapfrog: n_lf gradient passes
      for (int s = 0; s < n_lf; ++s) {
        const bool last = s == n_lf - 1;
        if (last) grad_pass<true>(sm, M, phase);
        else grad_pass<false>(sm, M, phase);
        const double scale = last ? half : eps;
        const int cu = sm.cur[oc];
        bool bad = false;
        double part = 0.0, part2 = 0.0;
#pragma unroll
        for (int j = 0; j < kOwn; ++j) {
          const int k = ok + 4 * j;
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
            const int k = ok + 4 * j;
            if (k < dim) {
              const double q = sm.qs[k * kLdS + oc] + eps * __ldg(M.inv_mass + k) * pown[j];
              bad |= !isfinite(q);
              sm.qs[k * kLdS + oc] = q;
            }
          }
        } else {
          sm.red[ok][oc] = part;
          sm.rs[ok * kLdS + oc] = part2;  // G no longer needed: reuse as prior partials
        }
        if (bad) sm.bad[oc] = 1;
        __syncthreads();
      }
      // -- energies, Metropolis (chain thread)
      if (is_chain) {
        const double k1 = sm.red[0][tid] + sm.red[1][tid] + sm.red[2][tid] + sm.red[3][tid];
        const double prior = sm.rs[0 * kLdS + tid] + sm.rs[1 * kLdS + tid] + sm.rs[2 * kLdS + tid] + sm.rs[3 * kLdS + tid];
        const double lp1 = sm.llp[0][tid] + sm.llp[1][tid] + prior;
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
            const int k = ok + 4 * j;
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
            sp += sigmoid_ll(M.y[i], eta);
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
