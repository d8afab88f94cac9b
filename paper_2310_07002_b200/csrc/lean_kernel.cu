// Lean sufficient-statistics HMC kernel (sm_100a, FP64) for the Gaussian models whose parameters are
// all global - grouped regression with one group (cfg1, cfg5: the J = 1 linear regression of
// SURVEY 8(d)) and seasonal AR (cfg4) - in the two modes that carry the work, Step-2 warm-up and
// Step-3 sampling (engine.cpp:296-381). One thread per chain holds the whole chain in registers for
// the launch: momentum, the drifted position and its gradient, the fold's training sums (its Gram
// matrix in a per-thread shared-memory column when d <= 6); the accepted state is read at each
// transition start and written on acceptance.
// The model is a compile-time shape (covariate count, AR order) so every parameter slot, mass and
// Gram index is static and the kernel stays a few thousand instructions (the general kernel
// carries every mode, family and probe and stalled on instruction fetch, profiles/r02_ncu_suff_*).
// Arithmetic is suff_pass's (gauss_impl.cuh): prepare / group_grad / global_grad on the masked sums
//   S_r = om.s - n off,  S_xr = (A om)[1..] - off s[1..],  S_rr = om^T A om - off (om.s + S_r),
// om = (1, -w), then the leapfrog (hmc.cpp:22-51), the energies and Metropolis test
// (hmc.cpp:53-99), log_pred (grouped_regression.cpp:124-163, seasonal_ar.cpp:107-115) and
// ScoreAccum::observe (accum.cpp:164-182). Probes, traces, HS/DSS and other shapes use the general
// kernels.
#include "gauss_impl.cuh"

namespace pcvg {

namespace {

constexpr int kLeanBlock = 128;

// Parameter dimension of the lean shapes: grouped J = 1 [alpha_0, beta_0..beta_{P-1}, mu_alpha,
// log sigma_alpha, log sigma_y] (NCM = P); seasonal [u_1..u_p, beta_0..beta_q, log sigma] (NCM = p+q).
template <int FAM, int NCM>
constexpr int lean_dim() { return FAM == kGrouped ? NCM + 4 : NCM + 2; }

// Global slot (gauss_impl.cuh gidx order) of parameter dimension d; -1 = the group intercept.
template <int FAM, int NCM, int PAR>
__device__ __forceinline__ constexpr int slot_of_dim(int d) {
  if constexpr (FAM == kGrouped) {
    return d == 0 ? -1 : (d <= NCM ? 2 + d : d - NCM - 1);
  } else {
    return d < PAR ? d + 2 : (d == PAR ? 0 : (d <= NCM ? d + 1 : 1));
  }
}

// Parameter dimension of global slot i (the inverse of slot_of_dim; gauss_impl.cuh gidx with the
// compile-time shape).
template <int FAM, int NCM, int PAR>
__device__ __forceinline__ constexpr int dim_of_slot(int i) {
  if constexpr (FAM == kGrouped) return i < 3 ? NCM + 1 + i : i - 2;
  else return i == 0 ? PAR : (i == 1 ? NCM + 1 : (i - 2 < PAR ? i - 2 : i - 1));
}

// Fold statistics of one chain: Gram entries (shared memory [e][thread] when small, else global
// through L1) and the group-0 training count / sums.
template <int E, bool SMEM>
struct LeanGram {
  const double* g;  // global [E] or shared column base (stride kLeanBlock)
  __device__ __forceinline__ double operator[](int e) const { return SMEM ? g[e * kLeanBlock] : __ldg(g + e); }
};

// The fold's Gram entries held in registers (few-chain launches, where registers are plentiful).
template <int E>
struct LeanGramReg {
  double a[E];
  __device__ __forceinline__ double operator[](int e) const { return a[e]; }
};

// prepare() (gauss_impl.cuh) with the compile-time shape: GEMM weights, variances, reciprocals.
template <int FAM, int NCM, int PAR>
__device__ __forceinline__ void lean_prepare(const ModelDev& M, const double* qG, Prep<NCM>& P, bool value) {
  if constexpr (FAM == kGrouped) {  // prepare(), grouped, with the compile-time covariate count
#pragma unroll
    for (int c = 0; c < NCM; ++c) P.w[c] = M.cmask[c] * qG[3 + c];
    const double sig_a = exp(qG[1]);
    const double sig_y = exp(qG[2]);
    P.va = sig_a * sig_a;
    P.v = sig_y * sig_y;
    P.off0 = 0.0;
    P.inv_va = 1.0 / P.va;
  } else {  // seasonal: rho(u) of the first PAR columns (seasonal_ar.cpp:37-46), dummies as they are
#pragma unroll
    for (int c = 0; c < NCM; ++c) {
      if (c < PAR) {
        const double w = logistic_fn(qG[2 + c]);
        P.w[c] = M.rho_sym ? 2.0 * w - 1.0 : 0.5 * (1.0 + w);
      } else {
        P.w[c] = qG[2 + c];
      }
    }
    P.off0 = qG[0];
    const double sigma = exp(qG[1]);
    P.v = sigma * sigma;
  }
  P.inv_v = 1.0 / P.v;
  if (value) P.logv = log(P.v);
}

// One gradient pass at the drifted position (qG, qa) (suff_pass, one lane): the masked sums from the
// fold statistics, the group and global gradients, and with VALUE the log joint with the reference's
// poisoning by a non-finite held-out row.
template <int FAM, int NCM, int PAR, bool VALUE, class GR>
__device__ __forceinline__ void lean_pass(const ModelDev& M, const GR& A, const double* s, double ng, int n_train,
                                          int ex0, int ex1, const double* qG, double qa, double* gG, double& ga,
                                          double& lp) {
  constexpr int NGM = FAM == kGrouped ? NCM + 3 : NCM + 2;
  constexpr int D = NCM + 1;
  Prep<NCM> P;
  lean_prepare<FAM, NCM, PAR>(M, qG, P, VALUE);
#define PCVG_OM(i) ((i) == 0 ? 1.0 : -P.w[(i) - 1])
  double q[D];
#pragma unroll
  for (int i = 0; i < D; ++i) q[i] = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      const double a = A[i * (i + 1) / 2 + j];
      q[i] = fma(a, PCVG_OM(j), q[i]);
      if (j < i) q[j] = fma(a, PCVG_OM(i), q[j]);
    }
  }
  GroupAcc G{0.0, 0.0, 0.0, 0.0};
  double om_u = 0.0;  // centred statistics: the offset shifts by om.ubar (suffstats.cpp)
#pragma unroll
  for (int i = 0; i < D; ++i) om_u = fma(PCVG_OM(i), M.su[i], om_u);
  const double off_raw = group_offset<FAM, NCM>(P, qa);
  const double off = off_raw - om_u;
  double ws = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) ws = fma(PCVG_OM(i), s[i], ws);
  const double srg = fma(-ng, off, ws);
  const double t2 = fma(off, ws + srg, 0.0);
  double sr_tot = 0.0;
  if constexpr (FAM == kGrouped) ga = group_grad<FAM, NCM, NGM, true>(P, qG, M, qa, srg, G);
  else sr_tot = srg;
  double quad = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) quad = fma(PCVG_OM(i), q[i], quad);
#undef PCVG_OM
  const double srr = quad - t2;
  double* sxr = q + 1;
#pragma unroll
  for (int k = 0; k < NCM; ++k) sxr[k] -= __dmul_rn(off, s[1 + k]);  // sum_g off_g s_g (one group)
  const double sr_all = 0.0 + srg;
#pragma unroll
  for (int k = 0; k < NCM; ++k) sxr[k] += M.su[1 + k] * sr_all;  // sum x r = sum x' r + xbar sum r
  if constexpr (VALUE) {
    bool poison = false;  // 0 * non-finite held-out term = NaN (grouped_regression.cpp:74-76)
    for (int tt = ex0; tt < ex1; ++tt) {
      const int i = __ldg(M.sex_rows + tt);
      double m = off_raw;
#pragma unroll
      for (int k = 0; k < NCM; ++k) m = fma(P.w[k], __ldg(M.x + static_cast<size_t>(k) * M.n + i), m);
      const double r = __ldg(M.y + i) - m;
      poison |= !isfinite(P.logv + r * r * P.inv_v);
    }
    global_grad<FAM, NCM, NGM, true>(M, P, qG, sxr, sr_tot, srr, G, n_train, gG, true, lp);
    if (poison) lp = CUDART_NAN;
  } else if constexpr (FAM == kGrouped) {  // global_grad (grouped_regression.cpp:109-121), gradient only
    const double ntr = static_cast<double>(n_train);
#pragma unroll
    for (int c = 0; c < NCM; ++c) gG[3 + c] = M.cmask[c] * dv<true>(sxr[c], P.v, P.inv_v) - qG[3 + c];
    gG[0] = G.a0 - qG[0];
    gG[1] = dv<true>(G.a1, P.va, P.inv_va) - M.J - P.va * 0.1 + 1.0;
    gG[2] = dv<true>(srr, P.v, P.inv_v) - ntr - P.v * 0.1 + 1.0;
  } else {  // seasonal_ar.cpp:79-105, gradient only
    const double ntr = static_cast<double>(n_train);
#pragma unroll
    for (int c = 0; c < NCM; ++c) {
      if (c < PAR) {
        const double w = logistic_fn(qG[2 + c]);
        const double dw = w * (1.0 - w);
        const double drho = M.rho_sym ? 2.0 * dw : 0.5 * dw;
        gG[2 + c] = dv<true>(sxr[c] * drho, P.v, P.inv_v) + (4.0 * (1.0 - w) - 4.0 * w + 1.0 - 2.0 * w);
      } else {
        gG[2 + c] = dv<true>(sxr[c], P.v, P.inv_v) - qG[2 + c];
      }
    }
    gG[0] = dv<true>(sr_tot, P.v, P.inv_v) - qG[0];
    gG[1] = dv<true>(srr, P.v, P.inv_v) - ntr - P.v + 1.0;
  }
}

// MINB: resident CTAs per SM the register allocation must allow (1 = full registers for latency-bound
// few-chain runs, the Gram in registers; 4 = 128 registers for many-chain runs that need
// more warps per SM, the Gram in shared memory when small).
template <int FAM, int NCM, int PAR, bool ASMEM, int MINB>
__global__ void __launch_bounds__(kLeanBlock, MINB) lean_kernel(ModelDev M, ChainsDev S, RunArgs A) {
  constexpr int NGM = FAM == kGrouped ? NCM + 3 : NCM + 2;
  constexpr int DIM = lean_dim<FAM, NCM>();
  constexpr int D = NCM + 1;
  constexpr int E = D * (D + 1) / 2;
  constexpr bool GRP = FAM == kGrouped;
  __shared__ double a_sm[ASMEM && !(MINB == 1 && E <= 21) ? E * kLeanBlock : 1];
  const int c = blockIdx.x * kLeanBlock + threadIdx.x;
  if (c >= S.nch) return;
  const int nch = S.nch;
  const int fold = S.fold0 + c / S.L;
  const int n_train = __ldg(M.n_train + fold);
  const size_t plane = static_cast<size_t>(DIM) * nch;
  const int cur = S.cur[c];

  // the fold's statistics: Gram (registers / a per-thread shared-memory column when small), count, sums
  constexpr bool AREG = MINB == 1 && E <= 21;
  const double* Aglob = M.sA + static_cast<size_t>(fold) * M.sdp;
  LeanGram<E, ASMEM && !AREG> Ag{Aglob};
  LeanGramReg<AREG ? E : 1> Ar;
  if constexpr (AREG) {
#pragma unroll
    for (int e = 0; e < E; ++e) Ar.a[e] = __ldg(Aglob + e);
  } else if constexpr (ASMEM) {
#pragma unroll
    for (int e = 0; e < E; ++e) a_sm[e * kLeanBlock + threadIdx.x] = __ldg(Aglob + e);
    Ag.g = a_sm + threadIdx.x;  // each thread reads only its own column: no barrier needed
  }
  double ng, s[D];
  {
    const int ov = __ldg(M.sov_ptr + fold), ov1 = __ldg(M.sov_ptr + fold + 1);
    const double* sp;
    if (ov < ov1 && __ldg(M.sov_g + ov) == 0) {
      ng = __ldg(M.sov_n + ov);
      sp = M.sov_s + static_cast<size_t>(ov) * D;
    } else {
      ng = __ldg(M.sgn);
      sp = M.sgs;
    }
#pragma unroll
    for (int i = 0; i < D; ++i) s[i] = __ldg(sp + i);
  }
  // inverse mass of global slot i / of the intercept (read through L1 where used)
  auto mG = [&](int i) { return __ldg(M.inv_mass + dim_of_slot<FAM, NCM, PAR>(i)); };
  const double ma = GRP ? __ldg(M.inv_mass) : 0.0;
  // the accepted position and its gradient live in plane `cur` (read at each transition start,
  // written on acceptance; the plane selector never flips in this kernel)
  auto at = [&](int d) { return cur * plane + static_cast<size_t>(d) * nch + c; };
  double lp0 = S.lp0[c];
  ChainRng R;
  R.init(S.seed, S.rng_stream[c], S.rng_pos[c], S.rng_cached[c], S.rng_has[c] != 0);
  const double eps = M.step, half = 0.5 * M.step;
  double em[NGM];  // eps * inverse mass of each slot (the drift factor, hmc.cpp:40)
#pragma unroll
  for (int i = 0; i < NGM; ++i) em[i] = eps * mG(i);
  const int n_lf = M.n_lf;
  const int ex0 = fold < M.K ? __ldg(M.sex_lo + fold) : 0, ex1 = fold < M.K ? __ldg(M.sex_hi + fold) : 0;
  int64_t div_count = 0;
  double warm = 0.0;

  for (int64_t it = 0; it < A.n_iters; ++it) {
    // momentum refresh in dimension order (the reference's draw order), global half kick
    double pG[NGM], pa = 0.0, k0G = 0.0, k0g = 0.0;
    // unrolled for the small grouped shapes; rolled for seasonal AR (DIM = 15: one inlined copy of
    // the Philox + Box-Muller code instead of 15 cut its kernel from ~20k to ~11k instructions and
    // cfg4 ran 4.6% faster; rolling the 9-dimensional grouped loop cost cfg5 7%)
    constexpr int kMomUnroll = DIM > 12 ? 1 : DIM;
#pragma unroll kMomUnroll
    for (int d = 0; d < DIM; ++d) {
      const double z = R.normal();
      const double p = z / sqrt(__ldg(M.inv_mass + d));  // = mG(slot_of_dim(d)), or ma for d = 0
      const int sl = slot_of_dim<FAM, NCM, PAR>(d);
      if (sl < 0) {
        pa = p;
      } else {
#pragma unroll
        for (int i = 0; i < NGM; ++i)
          if (i == sl) pG[i] = p;
      }
    }
#pragma unroll
    for (int i = 0; i < NGM; ++i) {
      k0G += mG(i) * pG[i] * pG[i];
      pG[i] = pG[i] + half * S.grad[at(dim_of_slot<FAM, NCM, PAR>(i))];
    }
    // leapfrog (hmc.cpp:22-51): first drift, then n_lf - 1 (gradient, full kick, drift) steps and
    // the value pass with the closing half kick; the intercept's half kick rides with the first drift
    // Finiteness (hmc.cpp:29-49 tests every position, gradient and momentum value along the
    // trajectory): a non-finite gradient makes the next momentum non-finite, and a non-finite
    // momentum or position stays non-finite under every later kick / drift (inf + finite = inf,
    // inf - inf = NaN), so testing the end point (q', p') is the same test.
    double qG[NGM], gG[NGM], qa = 0.0, ga = 0.0, lp1 = 0.0, k1g = 0.0;
#pragma unroll
    for (int i = 0; i < NGM; ++i) qG[i] = S.pos[at(dim_of_slot<FAM, NCM, PAR>(i))] + em[i] * pG[i];
    if constexpr (GRP) {
      k0g += ma * pa * pa;
      pa = pa + half * S.grad[at(0)];
      qa = S.pos[at(0)] + eps * ma * pa;
    }
    for (int st = 0; st + 1 < n_lf; ++st) {
      if constexpr (AREG) lean_pass<FAM, NCM, PAR, false>(M, Ar, s, ng, n_train, ex0, ex1, qG, qa, gG, ga, lp1);
      else lean_pass<FAM, NCM, PAR, false>(M, Ag, s, ng, n_train, ex0, ex1, qG, qa, gG, ga, lp1);
      if constexpr (GRP) {
        pa += eps * ga;
        qa = qa + eps * ma * pa;
      }
#pragma unroll
      for (int i = 0; i < NGM; ++i) {
        pG[i] += eps * gG[i];
        qG[i] = qG[i] + em[i] * pG[i];
      }
    }
    if constexpr (AREG) lean_pass<FAM, NCM, PAR, true>(M, Ar, s, ng, n_train, ex0, ex1, qG, qa, gG, ga, lp1);
    else lean_pass<FAM, NCM, PAR, true>(M, Ag, s, ng, n_train, ex0, ex1, qG, qa, gG, ga, lp1);
    double chk = 0.0;
    if constexpr (GRP) {
      pa += half * ga;
      k1g += ma * pa * pa;
      chk = fma(qa, 0.0, fma(pa, 0.0, chk));
    }
#pragma unroll
    for (int i = 0; i < NGM; ++i) {
      pG[i] += half * gG[i];
      chk = fma(qG[i], 0.0, fma(pG[i], 0.0, chk));
    }
    double k1G = 0.0;
#pragma unroll
    for (int i = 0; i < NGM; ++i) k1G += mG(i) * pG[i] * pG[i];
    const bool bad = isnan(chk) || fold == M.broken_fold;
    const double h0 = -lp0 + 0.5 * (k0g + k0G);
    const double h1 = bad ? CUDART_NAN : -lp1 + 0.5 * (k1g + k1G);
    const double dh = h1 - h0;
    const bool divergent = bad || isnan(dh) || (isfinite(dh) && fabs(dh) > 1000.0);
    if (divergent) {
      ++div_count;
    } else if (log(R.uniform()) < -dh) {
#pragma unroll
      for (int i = 0; i < NGM; ++i) {
        S.pos[at(dim_of_slot<FAM, NCM, PAR>(i))] = qG[i];
        S.grad[at(dim_of_slot<FAM, NCM, PAR>(i))] = gG[i];
      }
      if constexpr (GRP) {
        S.pos[at(0)] = qa;
        S.grad[at(0)] = ga;
      }
      lp0 = lp1;
    }
    // ---- log_pred at the current position (the fold's test rows; J = 1: the group is seen)
    double sp = 0.0;
    if (fold < M.K) {
      double xG[NGM];
#pragma unroll
      for (int i = 0; i < NGM; ++i) xG[i] = S.pos[at(dim_of_slot<FAM, NCM, PAR>(i))];
      Prep<NCM> P;
      prepare<FAM, NCM, NGM>(M, xG, P);
      const double v_pred = FAM == kSeasonal ? exp(2.0 * xG[1]) : P.v;
      const double off = FAM == kGrouped ? S.pos[at(0)] : P.off0;
      const int s0 = __ldg(M.fold_seg + fold), s1 = __ldg(M.fold_seg + fold + 1);
      for (int sg = s0; sg < s1; ++sg) {
        double a = 0.0;
        for (int tt = __ldg(M.seg_row + sg); tt < __ldg(M.seg_row + sg + 1); ++tt) {
          const int i = __ldg(M.seg_rows + tt);
          double m = off;
#pragma unroll
          for (int k = 0; k < NCM; ++k) m = fma(P.w[k], __ldg(M.x + static_cast<size_t>(k) * M.n + i), m);
          const double r = __ldg(M.y + i) - m;
          a += -0.5 * (kLog2Pi + log(v_pred) + r * r / v_pred);
        }
        sp += a;
      }
    }
    if (A.mode == kModeWarmup) warm += sp;
    else accum_observe(S.acc, c, nch, sp, A.iter0 + it, A.planned_n, A.D, A.b);
  }
  S.lp0[c] = lp0;
  S.rng_pos[c] = R.pos;
  S.rng_cached[c] = R.cached;
  S.rng_has[c] = R.has_cached ? 1 : 0;
  S.divergences[c] += div_count;
  if (A.mode == kModeWarmup) S.warm_sum[c] += warm;
}

template <int FAM, int NCM, int PAR>
cudaError_t launch_lean_t(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st) {
  const int grid = (S.nch + kLeanBlock - 1) / kLeanBlock;
  if (grid == 0) return cudaSuccess;
  constexpr bool ASMEM = (NCM + 1) * (NCM + 2) / 2 <= 28;  // Gram in shared memory (<= 28 KB per CTA)
  // (few-chain launches hold it in registers instead: lean_kernel's MINB = 1 instantiation)
  ++sampler_launch_count();
  static const int minb_env = std::getenv("PCVG_LEAN_MINB") ? std::atoi(std::getenv("PCVG_LEAN_MINB")) : 0;  // tuning
  // measured (profiles/r02_lean_*.log): cfg5's 1.6M chains are fastest at 4 CTAs/SM (128 registers,
  // some spills), cfg1 / cfg4 (400 / 800 chains, latency-bound) at full registers
  const int minb = minb_env ? minb_env : (grid >= 4 * device_sm_count() ? 4 : 1);
  if (minb == 4) lean_kernel<FAM, NCM, PAR, ASMEM, 4><<<grid, kLeanBlock, 0, st>>>(M, S, A);
  else lean_kernel<FAM, NCM, PAR, ASMEM, 1><<<grid, kLeanBlock, 0, st>>>(M, S, A);
  return cudaGetLastError();
}

}  // namespace

// The lean kernel when it covers this launch (warm-up / sampling, LogS, one lane per chain, a
// compiled shape, every test group seen), else cudaErrorNotSupported and the caller uses the
// general sufficient-statistics kernel.
cudaError_t launch_lean(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st) {
  if (!M.suff || (A.mode != kModeSample && A.mode != kModeWarmup) || S.X.kind != 0 || S.fold_override ||
      M.any_unseen || M.dim != (M.family == kGrouped ? M.nc + 4 : M.nc + 2))
    return cudaErrorNotSupported;
  if (M.family == kGrouped && M.J == 1) {
    switch (M.nc) {
      case 1: return launch_lean_t<kGrouped, 1, 0>(M, S, A, st);
      case 2: return launch_lean_t<kGrouped, 2, 0>(M, S, A, st);
      case 3: return launch_lean_t<kGrouped, 3, 0>(M, S, A, st);
      case 4: return launch_lean_t<kGrouped, 4, 0>(M, S, A, st);
      case 5: return launch_lean_t<kGrouped, 5, 0>(M, S, A, st);
      default: return cudaErrorNotSupported;
    }
  }
  if (M.family == kSeasonal && M.J == 0) {
    if (M.p == 1 && M.nc == 12) return launch_lean_t<kSeasonal, 12, 1>(M, S, A, st);
    if (M.p == 2 && M.nc == 13) return launch_lean_t<kSeasonal, 13, 2>(M, S, A, st);
    if (M.p == 1 && M.nc == 1) return launch_lean_t<kSeasonal, 1, 1>(M, S, A, st);
    if (M.p == 2 && M.nc == 2) return launch_lean_t<kSeasonal, 2, 2>(M, S, A, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace pcvg
