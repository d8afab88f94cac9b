// Per-chain setup and per-fold reduction kernels (sm_100a):
//  * init_chains   - Step 2 warm start (engine.cpp:296-309): stream keys, bank row drawn by
//                    CounterRng(seed, stream_key(ChainInit, m, k, c)).below(rows), fresh
//                    ChainSampling stream; one thread per chain.
//  * set_centers   - centering constants C_k = sum_c warm_c / (L N_wu) in chain order
//                    (engine.cpp:316-339); one thread per fold.
//  * fold_stats    - LogS fold score + R-hat of each fold from its L chain accumulators
//                    (scoring.cpp:10-62, diagnostics.cpp:11-44), same operation order as the
//                    reference; one thread per fold.
//  * extra_centers - HS / DSS centring vectors hs_c / pred_c = sum_c warm_c / (L N_wu) in chain
//                    order (engine.cpp:324-338); one block per fold.
//  * extra_merge   - per-fold WelfordDiag / WelfordAccumulator::merge over the L chains in chain
//                    order (engine.cpp:150-156, accum.cpp:28-34, 76-84); one block per fold.
#include <math_constants.h>

#include "device_common.cuh"
#include "score_extra.cuh"
#include "types.cuh"

namespace pcvg {

namespace {

__global__ void init_chains_kernel(ModelDev M, ChainsDev S, const double* bank, int64_t bank_rows) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= S.nch) return;
  const int fold = S.fold0 + c / S.L, chain = c % S.L;
  ChainRng init;
  init.init(S.seed, stream_key(2 /*ChainInit*/, S.stream_model, fold, chain), 0, 0.0, false);
  const uint64_t row = init.below(static_cast<uint64_t>(bank_rows));
  const size_t plane = static_cast<size_t>(M.dim) * S.nch;
  for (int d = 0; d < M.dim; ++d) {
    S.pos[static_cast<size_t>(d) * S.nch + c] = bank[row * M.dim + d];
    S.pos[plane + static_cast<size_t>(d) * S.nch + c] = 0.0;
  }
  S.cur[c] = 0;
  S.rng_stream[c] = stream_key(1 /*ChainSampling*/, S.stream_model, fold, chain);
  S.rng_pos[c] = 0;
  S.rng_cached[c] = 0.0;
  S.rng_has[c] = 0;
  S.divergences[c] = 0;
  S.warm_sum[c] = 0.0;
}

__global__ void reset_accum_kernel(ChainsDev S, int D, double* centers_per_fold) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= S.nch) return;
  const AccumDev& A = S.acc;
  A.u_x[c] = -CUDART_INF;
  A.u_x2[c] = -CUDART_INF;
  A.z_x[c] = -CUDART_INF;
  A.v_x[c] = -CUDART_INF;
  A.v_x2[c] = -CUDART_INF;
  A.committed[c] = 0;
  A.pending[c] = 0;
  A.count[c] = 0;
  A.faults[c] = 0;
  A.center[c] = centers_per_fold[c / S.L];
  for (int d = 0; d < D; ++d) {
    A.y_x[static_cast<size_t>(d) * S.nch + c] = 0.0;
    A.y_x2[static_cast<size_t>(d) * S.nch + c] = 0.0;
  }
}

__global__ void centers_kernel(ChainsDev S, int nfold, int64_t warmup, double* centers) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nfold) return;
  double c = 0.0;
  if (warmup > 0) {
    const double denom = static_cast<double>(S.L) * static_cast<double>(warmup);
    for (int ch = 0; ch < S.L; ++ch) c += S.warm_sum[k * S.L + ch] / denom;
  }
  centers[k] = c;
}

__device__ double logsumexp_dev(const double* v, int n) {  // math.hpp:24-32
  double m = -CUDART_INF;
  for (int i = 0; i < n; ++i)
    if (v[i] > m) m = v[i];
  if (m == -CUDART_INF) return -CUDART_INF;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += exp(v[i] - m);
  return m + log(s);
}

// rhat_from_sums (diagnostics.cpp:11-33) with the reference's rounding: explicit _rn products and
// sums keep nvcc from contracting dev*dev + b or (n-1)/n*w + b/n into FMAs.
__device__ bool rhat_from_sums_dev(const double* sx, const double* sxx, int l, int64_t n, double* rhat) {
  if (l < 2 || n < 2) return false;
  const double nd = static_cast<double>(n);
  double w = 0.0, grand = 0.0;
  for (int c = 0; c < l; ++c) {
    w = __dadd_rn(w, (sxx[c] - __dmul_rn(sx[c], sx[c]) / nd) / (nd - 1.0) / l);
    grand = __dadd_rn(grand, sx[c] / nd / l);
  }
  double bb = 0.0;
  for (int c = 0; c < l; ++c) {
    const double dev = sx[c] / nd - grand;
    bb = __dadd_rn(bb, __dmul_rn(dev, dev));
  }
  bb = __dmul_rn(bb, nd / (l - 1.0));
  if (!isfinite(w) || !isfinite(bb) || !(w > 0.0)) return false;
  *rhat = sqrt(__dadd_rn(__dmul_rn((nd - 1.0) / nd, w), bb / nd) / w);
  return true;
}

struct FoldOut {
  double *estimate, *log_f_hat, *mc, *naive, *ess, *rhat;
  int64_t* batches;
  int32_t* fault;
};

__global__ void fold_stats_kernel(ChainsDev S, int nfold, int64_t n, int b, int D, FoldOut out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nfold) return;
  const int l = S.L;
  const AccumDev& A = S.acc;
  const int c0 = k * l;
  const double ln = static_cast<double>(l) * static_cast<double>(n);
  double ux[64];
  bool fault = false;
  int64_t batches = 0;
  for (int c = 0; c < l; ++c) {
    ux[c] = A.u_x[c0 + c];
    fault = fault || A.faults[c0 + c] > 0;
    batches += A.committed[c0 + c];
  }
  const double lf = logsumexp_dev(ux, l) - log(ln);  // scoring.cpp:10-62
  double mc, naive, ess;
  if (lf == -CUDART_INF) {
    fault = true;
    mc = CUDART_INF;
    naive = CUDART_INF;
    ess = CUDART_NAN;
  } else {
    double sum_u2 = 0.0;
    for (int c = 0; c < l; ++c) sum_u2 += exp(A.u_x2[c0 + c] - 2.0 * lf);
    naive = ln > 1 ? (sum_u2 - ln) / (ln - 1.0) : 0.0;
    if (naive < 0.0) naive = 0.0;
    const int64_t a = A.committed[c0];
    if (batches >= 2 && a >= 1) {
      double ss = 0.0;
      for (int c = 0; c < l; ++c) {
        const double s2 = exp(A.v_x2[c0 + c] - 2.0 * lf);
        const double s1 = exp(A.v_x[c0 + c] - lf);
        ss += s2 - 2.0 * s1 + static_cast<double>(A.committed[c0 + c]);
      }
      mc = b * ss / (static_cast<double>(batches) - 1.0);
      if (mc < 0.0) mc = 0.0;
      ess = mc > 0.0 ? ln * naive / mc : CUDART_NAN;
    } else {
      mc = CUDART_NAN;
      ess = CUDART_NAN;
    }
  }
  // rhat_from_blocks (diagnostics.cpp:11-44)
  double rhat = CUDART_NAN;
  if (l >= 2 && n >= 2) {
    double sx[64], sxx[64];
    for (int c = 0; c < l; ++c) {
      double s = 0.0, s2 = 0.0;
      for (int d = 0; d < D; ++d) s += A.y_x[static_cast<size_t>(d) * S.nch + c0 + c];
      for (int d = 0; d < D; ++d) s2 += A.y_x2[static_cast<size_t>(d) * S.nch + c0 + c];
      sx[c] = s;
      sxx[c] = s2;
    }
    double rh;
    if (rhat_from_sums_dev(sx, sxx, l, n, &rh)) rhat = rh;
  }
  out.estimate[k] = lf;
  out.log_f_hat[k] = lf;
  out.mc[k] = mc;
  out.naive[k] = naive;
  out.ess[k] = ess;
  out.rhat[k] = rhat;
  out.batches[k] = batches;
  out.fault[k] = fault ? 1 : 0;
}

// Score streams: chain c feeds iterations [i0, i1) of its explicit stream s[c * stride + i] through
// accum_observe (accum.cpp:164-182) of a planned_n-iteration run.
__global__ void feed_streams_kernel(ChainsDev S, const double* s, int64_t stride, int64_t i0, int64_t i1,
                                    int64_t planned_n, int D, int b) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= S.nch) return;
  for (int64_t i = i0; i < i1; ++i) accum_observe(S.acc, c, S.nch, s[c * stride + i], i, planned_n, D, b);
}

__global__ void extra_centers_kernel(ExtraDev X, int L, int nfold, int64_t warmup) {
  const int k = blockIdx.x;
  if (k >= nfold) return;
  const int64_t len = extra_warm_len(X.kind, X.msize[k]);
  const double denom = static_cast<double>(L) * static_cast<double>(warmup);
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
    double c = 0.0;
    if (warmup > 0)
      for (int ch = 0; ch < L; ++ch) c += X.warm[X.wbase[k] + e * L + ch] / denom;
    X.center[X.cbase[k] + e] = c;
  }
}

// merged[base[k] / L + e] = sum over chains (in order) of entry e.
__global__ void extra_merge_kernel(ExtraDev X, int L, int nfold, double* merged) {
  const int k = blockIdx.x;
  if (k >= nfold) return;
  const int64_t len = extra_acc_len(X.kind, X.msize[k]);
  const double* A = X.acc + X.base[k];
  double* out = merged + X.base[k] / L;
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
    double s = A[e * L];
    for (int ch = 1; ch < L; ++ch) s += A[e * L + ch];
    out[e] = s;
  }
}

// Shuffle benchmark replicate maxima (diagnostics.cpp:76-101, engine.cpp:464-480) for the shard's
// folds of one model; thread = (replicate r, local fold k). The reference consumes replicate r's
// stream CounterRng(seed, stream_key(Benchmark, r, 0, 0)) sequentially, one below(L) per (model,
// non-failed fold, chain, block). below() takes one u64 per try and rejects only v >= L*floor(
// (2^64-1)/L) (probability < L/2^64), so without a rejection draw j of the stream is the u64 at
// words 2j, 2j+1: every item computes its draws at its global position and flags a rejection
// (the caller then runs the sequential host path for that replicate). R-hat > 0 always, so the
// maximum is kept as the bit pattern of a non-negative double (0 = no item) via atomicMax.
__global__ void bench_kernel(ChainsDev S, int nfold, const int64_t* item, int R, int sub_used,
                             int groups, int64_t n, unsigned long long* rep_max, int* reject) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int k = static_cast<int>(idx % nfold);
  const int r = static_cast<int>(idx / nfold);
  if (r >= R || item[k] < 0) return;
  const int l = S.L;
  const uint64_t L64 = static_cast<uint64_t>(l);
  const uint64_t bound = L64 * ((~0ull) / L64);
  const uint64_t stream = stream_key(6 /*Benchmark*/, static_cast<uint64_t>(r), 0, 0);
  const uint32_t k0 = static_cast<uint32_t>(S.seed), k1 = static_cast<uint32_t>(S.seed >> 32);
  uint64_t word = 2ull * static_cast<uint64_t>(item[k]) * L64 * static_cast<uint64_t>(groups);
  uint64_t blk_cached = ~0ull;
  uint4 buf = make_uint4(0, 0, 0, 0);
  bool rej = false;
  double sx[64], sxx[64];
  const size_t c0 = static_cast<size_t>(k) * l;
  for (int c = 0; c < l; ++c) {
    double a = 0.0, b = 0.0;
    for (int g = 0; g < groups; ++g, word += 2) {
      const uint64_t blk = word >> 2;
      if (blk != blk_cached) {
        buf = philox_block(blk, stream, k0, k1);
        blk_cached = blk;
      }
      const uint64_t v = (word & 2) ? (static_cast<uint64_t>(buf.z) | (static_cast<uint64_t>(buf.w) << 32))
                                    : (static_cast<uint64_t>(buf.x) | (static_cast<uint64_t>(buf.y) << 32));
      rej |= v >= bound;
      const size_t src = c0 + static_cast<size_t>(v % L64);
      // block g = sub-blocks [g*sub_used/groups, (g+1)*sub_used/groups) (one sub-block when equal)
      double ga = 0.0, gb = 0.0;
      for (int d = block_group_begin(g, sub_used, groups); d < block_group_begin(g + 1, sub_used, groups); ++d) {
        ga += S.acc.y_x[static_cast<size_t>(d) * S.nch + src];
        gb += S.acc.y_x2[static_cast<size_t>(d) * S.nch + src];
      }
      a += ga;
      b += gb;
    }
    sx[c] = a;
    sxx[c] = b;
  }
  if (rej) reject[r] = 1;
  double rh;
  if (!rhat_from_sums_dev(sx, sxx, l, n, &rh)) return;
  atomicMax(rep_max + r, static_cast<unsigned long long>(__double_as_longlong(rh)));
}

// Regrouped benchmark blocks: block g of chain c = sum of its sub-blocks [begin(g), begin(g + 1)) in
// order (the sums bench_kernel forms on the fly), written once so the R replicates each read
// `groups` values per chain instead of `sub_used`.
__global__ void regroup_kernel(const double* y_x, const double* y_x2, int nch, int sub_used, int groups,
                               double* g_x, double* g_x2) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nch) return;
  for (int g = 0; g < groups; ++g) {
    double a = 0.0, b = 0.0;
    for (int d = block_group_begin(g, sub_used, groups); d < block_group_begin(g + 1, sub_used, groups); ++d) {
      a += y_x[static_cast<size_t>(d) * nch + c];
      b += y_x2[static_cast<size_t>(d) * nch + c];
    }
    g_x[static_cast<size_t>(g) * nch + c] = a;
    g_x2[static_cast<size_t>(g) * nch + c] = b;
  }
}

}  // namespace

cudaError_t launch_regroup(const ChainsDev& S, int sub_used, int groups, double* g_x, double* g_x2,
                           cudaStream_t st) {
  if (S.nch == 0) return cudaSuccess;
  regroup_kernel<<<(S.nch + 255) / 256, 256, 0, st>>>(S.acc.y_x, S.acc.y_x2, S.nch, sub_used, groups, g_x, g_x2);
  return cudaGetLastError();
}

cudaError_t launch_bench(const ChainsDev& S, int nfold, const int64_t* item, int R, int sub_used,
                         int groups, int64_t n, unsigned long long* rep_max, int* reject,
                         cudaStream_t st) {
  if (nfold == 0 || R == 0) return cudaSuccess;
  if (S.L > 64) return cudaErrorInvalidValue;
  const int64_t total = static_cast<int64_t>(nfold) * R;
  bench_kernel<<<static_cast<unsigned>((total + 127) / 128), 128, 0, st>>>(S, nfold, item, R, sub_used,
                                                                         groups, n, rep_max, reject);
  return cudaGetLastError();
}

cudaError_t launch_extra_centers(const ChainsDev& S, int nfold, int64_t warmup, cudaStream_t st) {
  if (nfold == 0 || S.X.kind == 0) return cudaSuccess;
  extra_centers_kernel<<<nfold, 64, 0, st>>>(S.X, S.L, nfold, warmup);
  return cudaGetLastError();
}

cudaError_t launch_extra_merge(const ChainsDev& S, int nfold, double* merged, cudaStream_t st) {
  if (nfold == 0 || S.X.kind == 0) return cudaSuccess;
  extra_merge_kernel<<<nfold, 128, 0, st>>>(S.X, S.L, nfold, merged);
  return cudaGetLastError();
}

cudaError_t launch_feed_streams(const ChainsDev& S, const double* s, int64_t stride, int64_t i0, int64_t i1,
                                int64_t planned_n, int D, int b, cudaStream_t st) {
  feed_streams_kernel<<<(S.nch + 127) / 128, 128, 0, st>>>(S, s, stride, i0, i1, planned_n, D, b);
  return cudaGetLastError();
}

cudaError_t launch_init_chains(const ModelDev& M, const ChainsDev& S, const double* bank,
                               int64_t bank_rows, cudaStream_t st) {
  if (S.nch == 0) return cudaSuccess;
  init_chains_kernel<<<(S.nch + 255) / 256, 256, 0, st>>>(M, S, bank, bank_rows);
  return cudaGetLastError();
}

cudaError_t launch_centers(const ChainsDev& S, int nfold, int64_t warmup, double* centers,
                           int D, cudaStream_t st) {
  if (nfold > 0) centers_kernel<<<(nfold + 127) / 128, 128, 0, st>>>(S, nfold, warmup, centers);
  if (S.nch > 0) reset_accum_kernel<<<(S.nch + 255) / 256, 256, 0, st>>>(S, D, centers);
  return cudaGetLastError();
}

cudaError_t launch_fold_stats(const ChainsDev& S, int nfold, int64_t n, int b, int D,
                              double* estimate, double* log_f_hat, double* mc, double* naive,
                              double* ess, double* rhat, int64_t* batches, int32_t* fault,
                              cudaStream_t st) {
  if (nfold == 0) return cudaSuccess;
  if (S.L > 64) return cudaErrorInvalidValue;
  FoldOut o{estimate, log_f_hat, mc, naive, ess, rhat, batches, fault};
  fold_stats_kernel<<<(nfold + 127) / 128, 128, 0, st>>>(S, nfold, n, b, D, o);
  return cudaGetLastError();
}

}  // namespace pcvg
