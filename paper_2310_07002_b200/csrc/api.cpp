// libpcvg.so: the C ABI (include/pcvg.h) over the B200 kernels.
//
// Host driver for Steps 2-4 of the reference engine (engine.cpp:257-483): model upload in the
// device layout, chain-state allocation, the warm-up / sampling launches, per-fold reductions and
// the Step-4 merge (compute_stats, failed folds, shuffle benchmark, verdict). Every preconditions
// check of the reference is repeated here and returned as a status code (errors.hpp taxonomy).
// There is no CPU fallback: without a working CUDA device every device entry point returns
// PCVG_CUDA_ERROR.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/pcvg.h"
#include "host_common.hpp"
#include "score_extra.cuh"
#include "suffstats.hpp"
#include "types.cuh"

namespace pcvg {

// kernels (gauss_kernel.cu, glm_kernel.cu, chain_kernels.cu)
int gauss_lanes_per_chain(const ModelDev& M, int nch);
int suff_lanes_per_chain(const ModelDev& M, int nch);
cudaError_t launch_gauss(const ModelDev& M, const ChainsDev& S, const RunArgs& A, int T, cudaStream_t st);
int glm_width(int family, int J, int nc);
int glm_cluster_size(int n, int kp, int nch);
cudaError_t launch_glm(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st);
cudaError_t launch_lean(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st);
void glm_multicluster_scratch(int kp, int nch, size_t* part_doubles, size_t* counters);
cudaError_t launch_glm32(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st);
size_t glm32_scratch_doubles(int nch);
size_t glm32_image_bytes(int64_t n);
void glm32_tile_image(const double* xr, int kp, const double* y, const int* key, int64_t n, unsigned char* out);
cudaError_t launch_init_chains(const ModelDev& M, const ChainsDev& S, const double* bank,
                               int64_t bank_rows, cudaStream_t st);
cudaError_t launch_centers(const ChainsDev& S, int nfold, int64_t warmup, double* centers, int D,
                           cudaStream_t st);
cudaError_t launch_fold_stats(const ChainsDev& S, int nfold, int64_t n, int b, int D,
                              double* estimate, double* log_f_hat, double* mc, double* naive,
                              double* ess, double* rhat, int64_t* batches, int32_t* fault,
                              cudaStream_t st);
cudaError_t launch_feed_streams(const ChainsDev& S, const double* s, int64_t stride, int64_t i0, int64_t i1,
                                int64_t planned_n, int D, int b,
                                cudaStream_t st);
cudaError_t launch_extra_centers(const ChainsDev& S, int nfold, int64_t warmup, cudaStream_t st);
cudaError_t launch_extra_merge(const ChainsDev& S, int nfold, double* merged, cudaStream_t st);
cudaError_t launch_regroup(const ChainsDev& S, int sub_used, int groups, double* g_x, double* g_x2, cudaStream_t st);
cudaError_t launch_bench(const ChainsDev& S, int nfold, const int64_t* item, int R, int sub_used,
                         int groups, int64_t n, unsigned long long* rep_max, int* reject,
                         cudaStream_t st);
// host_folds.cpp
void rng_sequence(uint64_t, uint64_t, int32_t, uint64_t, const char*, const uint64_t*, int64_t, double*);
void make_loo(int64_t, int32_t*, int32_t*);
void make_logo(const pcvg_dataset*, int32_t*, int32_t*);
void make_kfold(int64_t, int32_t, uint64_t, int32_t*);
void make_time_blocks(const pcvg_dataset*, int32_t, int32_t*);
void make_hv_block(const pcvg_dataset*, int32_t, int64_t, int64_t*);
void make_hv_racine(const pcvg_dataset*, int64_t, int64_t, int64_t*);
void simulate_linreg(int64_t, int32_t, uint64_t, double*, double*, int32_t*);
void simulate_logistic(int64_t, int32_t, uint64_t, double*, double*);
// stats.cpp
void merge_stats(int32_t n_models, int32_t K, const pcvg_run_config* cfg, int64_t iter_count,
                 int32_t final_checkpoint, const pcvg_fold_table* folds, const double* y_x,
                 const double* y_x2, int sub_used, pcvg_report* rep, const double* bench_max);
void bench_shard(int32_t nm, int32_t nfold, int32_t l, int32_t D_stride, int32_t sub_used, int32_t groups, int64_t n,
                 uint64_t seed, int32_t R, const double* y_x, const double* y_x2,
                 const int32_t* failed, int64_t nonfailed_before, int64_t nonfailed_total,
                 double* rep_max, int32_t* needs_host);
double hs_fold_estimate(const double* a_x, const double* center, int m, int64_t count);
bool dss_fold_estimate(const double* merged, const double* center, const double* y_test, int m,
                       int64_t count, double* score, int* ridged);

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(PCVG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffers come from the device's stream-ordered memory pool (cudaMallocAsync / cudaFreeAsync on
// the owning context's stream), which keeps its memory mapped between uses: a context teardown returns
// ~300 MB of chain state to the pool in milliseconds, where cudaFree unmapped it in 2 s
// (profiles/r02_teardown.log), and the next context on the device reuses it.
thread_local cudaStream_t g_alloc_stream = nullptr;  // the calling context's stream (set by guarded())

// Host-to-device copies and clears, ordered with every later kernel. A plain cudaMemcpy from pageable
// host memory may return before its DMA has landed and cudaMemset is asynchronous, both on the legacy
// stream, which the contexts' non-blocking streams do not wait for: a kernel on the context's stream
// could read a buffer before its upload or clear completed (an intermittent acceptance-test failure:
// a score-stream run read part of its streams before they arrived). Here the copy / clear runs on the
// context's stream and the host waits for it, so any stream sees the data afterwards.
void h2d(void* dst, const void* src, size_t bytes, cudaStream_t st = g_alloc_stream) {
  if (!bytes) return;
  ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), "upload");
  ck(cudaStreamSynchronize(st), "upload");
}
void dzero(void* p, size_t bytes, cudaStream_t st = g_alloc_stream) {
  if (!bytes) return;
  ck(cudaMemsetAsync(p, 0, bytes, st), "memset");
  ck(cudaStreamSynchronize(st), "memset");
}

void retain_pool_memory() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> g(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done.push_back(dev);
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t st = nullptr;  // stream the buffer was allocated on; freed in its order
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  void alloc(size_t count) {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    n = count;
    st = g_alloc_stream;
    if (count) {
      ck(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, st), "cudaMallocAsync");
      ck(cudaStreamSynchronize(st), "alloc");  // usable from any stream (synchronous copies) from here
    }
  }
  void upload(const std::vector<T>& v) {
    alloc(v.size());
    if (!v.empty()) h2d(p, v.data(), sizeof(T) * v.size(), st);
  }
  std::vector<T> download(cudaStream_t s) const {
    std::vector<T> v(n);
    if (n) {
      ck(cudaMemcpyAsync(v.data(), p, sizeof(T) * n, cudaMemcpyDeviceToHost, s), "download");
      ck(cudaStreamSynchronize(s), "sync");
    }
    return v;
  }
};

struct HostModel {
  int family = 0;
  int64_t n = 0;
  int K = 0;
  int J = 0, ng = 0, dim = 0, nc = 0;
  int model_id = 0;
  bool hv = false;
  std::vector<int> perm;  // device row -> original row
  std::vector<int> fold_seg, seg_row, seg_rows;  // host copies of the test layout
  std::vector<double> y_host;                    // y in device row order (test_values)
  DevBuf<double> y, x, xr, inv_mass, bank;
  DevBuf<int> key, grp_ptr, lo, hi, ntrain, fseg, sgroup, sunseen, srow, srows;
  DevBuf<double> yb, xb;         // group-batched layout (ModelDev::nb > 0)
  DevBuf<unsigned char> x32;     // logistic FP32 variant tile images
  DevBuf<int> keyb, bgroup, boff, tfirst, tr0, trows, bkey, bgrows, buni;
  DevBuf<double> sA, sgn, sgs, sov_n, sov_s, sgA, sov_A;  // fold sufficient statistics (suffstats.cpp)
  DevBuf<int> sov_ptr, sov_g, sex_lo, sex_hi, sex_rows, sex_grp;
  mutable DevBuf<double> g32;  // FP32 variant G scratch (grown on first use, per model)
  mutable DevBuf<double> glm_part;      // few-chain multi-cluster GLM launches: cluster partials
  mutable DevBuf<unsigned int> glm_cnt;  // and per-tile arrival counters
  int64_t bank_rows = 0;
  ModelDev md{};
};

struct ChainSet {
  int nch = 0, dim = 0, D = 0;
  DevBuf<double> pos, grad, wp, lp0, warm, cached;
  DevBuf<int8_t> cur, has;
  DevBuf<uint64_t> stream, rpos;
  DevBuf<int64_t> div;
  DevBuf<int> fold_override;
  // accumulators
  DevBuf<double> u_x, u_x2, z_x, v_x, v_x2, center, y_x, y_x2;
  DevBuf<int64_t> committed, count, faults;
  DevBuf<int32_t> pending;
  // HS / DSS state (ExtraDev, types.cuh)
  int xkind = 0;
  std::vector<int> xm;
  std::vector<int64_t> xbase_h, xwbase_h, xcbase_h;
  DevBuf<int> xmsize;
  DevBuf<int64_t> xbase, xwbase, xcbase;
  DevBuf<double> xacc, xwarm, xdev, xcenter;

  void alloc(int n, int d, int blocks) {
    nch = n;
    dim = d;
    D = blocks;
    pos.alloc(2 * static_cast<size_t>(d) * n);
    grad.alloc(2 * static_cast<size_t>(d) * n);
    wp.alloc(static_cast<size_t>(d) * n);
    lp0.alloc(n);
    warm.alloc(n);
    cached.alloc(n);
    cur.alloc(n);
    has.alloc(n);
    stream.alloc(n);
    rpos.alloc(n);
    div.alloc(n);
    u_x.alloc(n);
    u_x2.alloc(n);
    z_x.alloc(n);
    v_x.alloc(n);
    v_x2.alloc(n);
    center.alloc(n);
    y_x.alloc(static_cast<size_t>(std::max(blocks, 1)) * n);
    y_x2.alloc(static_cast<size_t>(std::max(blocks, 1)) * n);
    committed.alloc(n);
    count.alloc(n);
    faults.alloc(n);
    pending.alloc(n);
  }
  ChainsDev view(int L, int fold0, uint64_t seed, uint64_t stream_model) const {
    ChainsDev s{};
    s.nch = nch;
    s.L = L;
    s.fold0 = fold0;
    s.fold_override = fold_override.p;
    s.seed = seed;
    s.stream_model = stream_model;
    s.pos = pos.p;
    s.grad = grad.p;
    s.wp = wp.p;
    s.lp0 = lp0.p;
    s.cur = cur.p;
    s.rng_stream = stream.p;
    s.rng_pos = rpos.p;
    s.rng_cached = cached.p;
    s.rng_has = has.p;
    s.divergences = div.p;
    s.warm_sum = warm.p;
    s.acc = AccumDev{u_x.p, u_x2.p, z_x.p, v_x.p, v_x2.p, committed.p, pending.p, count.p, faults.p, center.p, y_x.p, y_x2.p};
    s.X = ExtraDev{xkind, xmsize.p, xbase.p, xwbase.p, xcbase.p, xacc.p, xwarm.p, xdev.p, xcenter.p};
    return s;
  }
};

}  // namespace
}  // namespace pcvg

using namespace pcvg;

struct pcvg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // second candidate model runs concurrently (engine.cpp:342)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evj = nullptr;
  std::vector<std::unique_ptr<HostModel>> models;
  std::string err;
  // run state
  bool begun = false;
  pcvg_run_config cfg{};
  int b = 0, fb = 0, fe = 0;
  std::vector<std::unique_ptr<ChainSet>> chains;
  std::vector<std::unique_ptr<DevBuf<double>>> centers;
  std::vector<std::vector<int64_t>> div_base;
  int64_t iters_done = 0;
  double last_ms = 0.0, warm_ms = 0.0, sample_ms = 0.0;
  int64_t launches = 0;
  int policy = PCVG_KERNEL_AUTO;
  // score-stream runs (pcvg_run_streams): chains observe given log_pred streams instead of sampling
  bool stream_mode = false;
  DevBuf<double> stream_scores;  // [K*L][iters]
};

namespace {

thread_local std::string g_last_error;

template <class F>
int32_t guarded(pcvg_ctx* ctx, F&& f) {
  struct StreamScope {  // device buffers allocated by this call belong to the context's stream
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
    ~StreamScope() { g_alloc_stream = prev; }
  } scope(ctx ? ctx->stream : nullptr);
  try {
    f();
    return PCVG_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    if (ctx) ctx->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    if (ctx) ctx->err = e.what();
    return PCVG_INVALID_INPUT;
  }
}

int n_groups(const pcvg_dataset* d) {
  int j = 0;
  for (int64_t i = 0; i < d->n_obs; ++i) j = std::max(j, d->group_id[i] + 1);
  return j;
}

// Device layout of one model.
std::unique_ptr<HostModel> build_model(const pcvg_dataset* d, const pcvg_folds* f,
                                       const pcvg_model_spec* s, const pcvg_kernel* kp,
                                       const double* bank, int64_t bank_rows, int model_id) {
  if (!d || !f || !s || !kp) throw Error(PCVG_INVALID_INPUT, "null descriptor");
  if (d->n_obs < 1) throw Error(PCVG_INVALID_INPUT, "dataset is empty");
  if (d->n_obs > (1LL << 30)) throw Error(PCVG_INVALID_INPUT, "dataset too large for int32 row ids");
  auto hm = std::make_unique<HostModel>();
  HostModel& m = *hm;
  const int64_t n = d->n_obs;
  m.family = s->family;
  m.n = n;
  m.K = f->K;
  m.model_id = model_id;
  m.hv = f->intervals != nullptr;
  if (!f->test_index && !f->intervals) throw Error(PCVG_INVALID_INPUT, "folds need test_index or intervals");
  if (f->K < 1) throw Error(PCVG_INVALID_INPUT, "fold count must be at least 1");
  const bool hier = s->family == PCVG_FAMILY_GROUPED || s->family == PCVG_FAMILY_RADON ||
                    s->family == PCVG_FAMILY_RAT_GROWTH;
  if (d->group_id) {  // Dataset::validate (dataset.cpp:19-39)
    std::vector<char> seen(n_groups(d), 0);
    for (int64_t i = 0; i < n; ++i) {
      if (d->group_id[i] < 0) throw Error(PCVG_INVALID_INPUT, "group ids must be 0-based");
      seen[d->group_id[i]] = 1;
    }
    for (char c : seen)
      if (!c) throw Error(PCVG_INVALID_INPUT, "group ids must form a contiguous 0..J-1 range");
  }
  switch (s->family) {
    case PCVG_FAMILY_GROUPED:
      if (!d->group_id) throw Error(PCVG_INVALID_INPUT, "grouped regression needs a group column");
      if (d->n_cov > 8) throw Error(PCVG_INVALID_INPUT, "grouped family supports at most 8 covariates on device");
      m.J = n_groups(d);
      m.nc = d->n_cov;
      m.ng = d->n_cov + 3;
      break;
    case PCVG_FAMILY_RADON:
      if (!d->group_id || d->n_cov < 1)
        throw Error(PCVG_INVALID_INPUT, "radon-style model needs a group column and a floor covariate");
      m.J = n_groups(d);
      m.nc = 1;
      m.ng = 4;
      break;
    case PCVG_FAMILY_SEASONAL_AR:
      if (s->ar_order < 1) throw Error(PCVG_INVALID_INPUT, "AR order must be at least 1");
      if (s->dummies < 0) throw Error(PCVG_INVALID_INPUT, "dummy count must be non-negative");
      if (d->n_cov < s->ar_order + s->dummies)
        throw Error(PCVG_INVALID_INPUT, "dataset must carry lag and dummy covariates");
      if (s->ar_order + s->dummies > 13) throw Error(PCVG_INVALID_INPUT, "seasonal family supports p + q <= 13 on device");
      m.J = 0;
      m.nc = s->ar_order + s->dummies;
      m.ng = m.nc + 2;
      break;
    case PCVG_FAMILY_LOGISTIC:
      if (d->n_cov > 51) throw Error(PCVG_INVALID_INPUT, "logistic family supports at most 51 covariates on device");
      m.J = 0;
      m.nc = d->n_cov;
      m.ng = d->n_cov + 1;
      break;
    case PCVG_FAMILY_RAT_GROWTH:  // rat_growth.cpp:13-48
      if (!d->group_id || d->n_cov < 1)
        throw Error(PCVG_INVALID_INPUT, "growth model needs a group column and a time covariate");
      m.J = n_groups(d);
      m.nc = 1;
      m.ng = s->per_subject_slope ? 5 : 4;
      if (m.J > 32 * kMaxBatches)
        throw Error(PCVG_INVALID_INPUT, "growth model supports at most 512 subjects on device");
      break;
    default:
      throw Error(PCVG_INVALID_INPUT, "unknown model family");
  }
  const int gdims = (s->family == PCVG_FAMILY_RAT_GROWTH && s->per_subject_slope) ? 2 : 1;
  m.dim = m.J * gdims + m.ng;
  if (!kp->inv_mass_diag) throw Error(PCVG_INVALID_INPUT, "inverse mass diagonal missing");
  if (kp->n_leapfrog < 1) throw Error(PCVG_INVALID_INPUT, "n_leapfrog must be >= 1");
  for (int i = 0; i < m.dim; ++i)
    if (!(kp->inv_mass_diag[i] > 0.0)) throw Error(PCVG_INVALID_INPUT, "inverse mass diagonal must be positive");
  if (!bank || bank_rows < 1) throw Error(PCVG_INVALID_INPUT, "empty full-data draw bank");

  // time rank (hv folds)
  std::vector<int64_t> rank;
  if (m.hv) {
    if (!d->time_index) throw Error(PCVG_INVALID_INPUT, "hv-block folds need a time column");
    const auto order = time_order(d->time_index, n);
    rank.assign(n, 0);
    for (int64_t r = 0; r < n; ++r) rank[order[r]] = r;
  }
  // fold validation (folds.cpp:25-41 / hv analogue)
  std::vector<int64_t> test_count(m.K, 0);
  if (!m.hv) {
    for (int64_t i = 0; i < n; ++i) {
      const int t = f->test_index[i];
      if (t < 0 || t >= m.K) throw Error(PCVG_INVALID_INPUT, "test_index out of range");
      ++test_count[t];
    }
    for (int k = 0; k < m.K; ++k) {
      if (test_count[k] == 0) throw Error(PCVG_INVALID_INPUT, "fold " + std::to_string(k) + " has empty test set");
      if (test_count[k] == n) throw Error(PCVG_INVALID_INPUT, "fold " + std::to_string(k) + " has empty training set");
    }
  } else {
    for (int k = 0; k < m.K; ++k) {
      const int64_t* iv = f->intervals + 4 * k;
      if (!(0 <= iv[2] && iv[2] <= iv[0] && iv[0] < iv[1] && iv[1] <= iv[3] && iv[3] <= n))
        throw Error(PCVG_INVALID_INPUT, "hv-block fold " + std::to_string(k) + " has a malformed interval");
      if (iv[3] - iv[2] >= n) throw Error(PCVG_INVALID_INPUT, "fold " + std::to_string(k) + " has empty training set");
    }
  }

  // device row order: group-major for hierarchical families (stable)
  m.perm.resize(n);
  std::iota(m.perm.begin(), m.perm.end(), 0);
  std::vector<int> grp_ptr;
  if (hier) {
    std::stable_sort(m.perm.begin(), m.perm.end(),
                     [&](int a, int b) { return d->group_id[a] < d->group_id[b]; });
    grp_ptr.assign(m.J + 1, 0);
    for (int64_t i = 0; i < n; ++i) ++grp_ptr[d->group_id[i] + 1];
    for (int g = 0; g < m.J; ++g) grp_ptr[g + 1] += grp_ptr[g];
  }
  std::vector<int> inv(n);
  for (int64_t r = 0; r < n; ++r) inv[m.perm[r]] = static_cast<int>(r);

  // Tensor-core (GLM) path: no group effects beyond one intercept (glm_kernel.cu).
  const int glm_kp = glm_width(s->family, m.J, m.nc);
  const int64_t n_pad = glm_kp > 0 ? ((n + 255) / 256) * 256 : n;
  std::vector<double> y(n_pad, 0.0);
  std::vector<int> key(n_pad, -1);
  std::vector<double> xc(static_cast<size_t>(std::max(m.nc, 1)) * n, 0.0);
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = m.perm[r];
    y[r] = d->y[i];
    key[r] = m.hv ? static_cast<int>(rank[i]) : f->test_index[i];
    for (int c = 0; c < m.nc; ++c) xc[static_cast<size_t>(c) * n + r] = d->x[i * d->n_cov + c];
  }
  m.y.upload(y);
  m.key.upload(key);
  m.x.upload(xc);
  int nc_pad = 0;
  if (glm_kp > 0) {
    nc_pad = glm_kp;
    std::vector<double> xr(static_cast<size_t>(n_pad) * nc_pad, 0.0);
    for (int64_t r = 0; r < n; ++r) {
      xr[r * nc_pad] = 1.0;
      for (int c = 0; c < m.nc; ++c) xr[r * nc_pad + 1 + c] = d->x[m.perm[r] * d->n_cov + c];
    }
    m.xr.upload(xr);
    if (s->family == PCVG_FAMILY_LOGISTIC && m.nc + 1 <= 56) {  // FP32 (tcgen05 TF32) variant
      std::vector<unsigned char> img(glm32_image_bytes(n));
      glm32_tile_image(xr.data(), nc_pad, y.data(), key.data(), n, img.data());
      m.x32.upload(img);
    }
  }
  m.grp_ptr.upload(hier ? grp_ptr : std::vector<int>{0});

  // Group-batched layout for the hierarchical kernel (types.cuh): groups sorted by row count
  // (descending, stable), 32 per batch; batch b is padded to its largest group.
  int nb = 0, bstride = 0, ntile = 0, rt = 0, bkey_uniform = 0, ring = 0;
  if (hier && m.J > 1 && m.J <= 32 * kMaxBatches) {
    std::vector<int> order(m.J);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return grp_ptr[a + 1] - grp_ptr[a] > grp_ptr[b + 1] - grp_ptr[b];
    });
    nb = (m.J + 31) / 32;
    std::vector<int> bgroup(static_cast<size_t>(nb) * 32, -1), boff(nb + 1, 0);
    for (int b = 0; b < nb; ++b) {
      int rows = 0;
      for (int i = 0; i < 32 && 32 * b + i < m.J; ++i) {
        const int g = order[32 * b + i];
        bgroup[32 * b + i] = g;
        rows = std::max(rows, grp_ptr[g + 1] - grp_ptr[g]);
      }
      boff[b + 1] = boff[b] + rows;
    }
    bstride = boff[nb];
    const size_t tot = static_cast<size_t>(bstride) * 32;
    std::vector<double> ybv(tot, 0.0), xbv(static_cast<size_t>(std::max(m.nc, 1)) * tot, 0.0);
    std::vector<int> kbv(tot, -1);
    for (int b = 0; b < nb; ++b)
      for (int i = 0; i < 32; ++i) {
        const int g = bgroup[32 * b + i];
        if (g < 0) continue;
        for (int r = grp_ptr[g]; r < grp_ptr[g + 1]; ++r) {
          const size_t idx = static_cast<size_t>(boff[b] + (r - grp_ptr[g])) * 32 + i;
          ybv[idx] = y[r];
          kbv[idx] = key[r];
          for (int c = 0; c < m.nc; ++c) xbv[c * tot + idx] = xc[static_cast<size_t>(c) * n + r];
        }
      }
    m.yb.upload(ybv);
    m.xb.upload(xbv);
    m.keyb.upload(kbv);
    m.bgroup.upload(bgroup);
    m.boff.upload(boff);
    // per-slot group key when every group's rows share one key (LOGO-style folds)
    std::vector<int> bkey(static_cast<size_t>(nb) * 32, -1), bgrows(static_cast<size_t>(nb) * 32, 0);
    bkey_uniform = 1;
    for (int s2 = 0; s2 < nb * 32; ++s2) {
      const int g = bgroup[s2];
      if (g < 0) continue;
      bkey[s2] = key[grp_ptr[g]];
      bgrows[s2] = grp_ptr[g + 1] - grp_ptr[g];
      for (int r = grp_ptr[g]; r < grp_ptr[g + 1]; ++r)
        if (key[r] != bkey[s2]) bkey_uniform = 0;
    }
    m.bkey.upload(bkey);
    m.bgrows.upload(bgrows);
    std::vector<int> buni(nb, 1);
    for (int b = 0; b < nb; ++b)
      for (int i = 0; i < 32; ++i)
        if (bgroup[32 * b + i] >= 0 && bgrows[32 * b + i] != boff[b + 1] - boff[b]) buni[b] = 0;
    m.buni.upload(buni);
    // row tiles: staged through a shared-memory ring (<= 16 KB per slot) or, ring off, one tile
    // per batch read through L1 (PCVG_BATCH_RING=0/1 overrides; default on)
    const char* ring_env = std::getenv("PCVG_BATCH_RING");
    ring = ring_env ? std::atoi(ring_env) != 0 : 1;
    rt = ring ? std::max(1, 16384 / (32 * (8 + 8 * std::max(m.nc, 1) + (bkey_uniform ? 0 : 4)))) : 1 << 30;
    std::vector<int> tfirst(nb + 1, 0), tr0, trows;
    for (int b = 0; b < nb; ++b) {
      for (int r = boff[b]; r < boff[b + 1]; r += rt) {
        tr0.push_back(r);
        trows.push_back(std::min(rt, boff[b + 1] - r));
      }
      tfirst[b + 1] = static_cast<int>(tr0.size());
    }
    ntile = static_cast<int>(tr0.size());
    m.tfirst.upload(tfirst);
    m.tr0.upload(tr0.empty() ? std::vector<int>{0} : tr0);
    m.trows.upload(trows.empty() ? std::vector<int>{0} : trows);
  }

  // fold tables (index K = sentinel: nothing held out)
  std::vector<int> lo(m.K + 1, 0), hi(m.K + 1, 0), ntr(m.K + 1, static_cast<int>(n));
  for (int k = 0; k < m.K; ++k) {
    if (m.hv) {
      lo[k] = static_cast<int>(f->intervals[4 * k + 2]);
      hi[k] = static_cast<int>(f->intervals[4 * k + 3]);
      ntr[k] = static_cast<int>(n - (hi[k] - lo[k]));
    } else {
      lo[k] = k;
      hi[k] = k + 1;
      ntr[k] = static_cast<int>(n - test_count[k]);
    }
  }
  m.lo.upload(lo);
  m.hi.upload(hi);
  m.ntrain.upload(ntr);

  // fold sufficient statistics for the Gaussian linear families (suffstats.cpp)
  int suff = 0;
  SuffStats ss;
  const bool per_subject = s->family == PCVG_FAMILY_RAT_GROWTH && s->per_subject_slope;
  if ((s->family == PCVG_FAMILY_GROUPED || s->family == PCVG_FAMILY_RADON || s->family == PCVG_FAMILY_SEASONAL_AR ||
       s->family == PCVG_FAMILY_RAT_GROWTH) &&
      build_suffstats(n, m.nc, m.J, y.data(), xc.data(), key.data(), hier ? grp_ptr.data() : nullptr, m.K,
                      lo.data(), hi.data(), ss, per_subject)) {
    suff = 1;
    m.sA.upload(ss.A);
    m.sgn.upload(ss.gn);
    m.sgs.upload(ss.gs);
    m.sov_ptr.upload(ss.ov_ptr);
    m.sov_g.upload(ss.ov_g);
    m.sov_n.upload(ss.ov_n);
    m.sov_s.upload(ss.ov_s);
    m.sex_lo.upload(ss.ex_lo);
    m.sex_hi.upload(ss.ex_hi);
    m.sex_rows.upload(ss.ex_rows);
    m.sex_grp.upload(ss.ex_grp);
    if (per_subject) {
      m.sgA.upload(ss.gA);
      m.sov_A.upload(ss.ov_A);
    }
  }

  // test segments (fold_meta_, grouped_regression.cpp:27-47): test rows grouped by group in
  // increasing group order, rows increasing within a group; unseen = no training row in group.
  const int Jg = hier ? m.J : 1;
  std::vector<int64_t> gsize(Jg, 0);
  for (int64_t i = 0; i < n; ++i) gsize[hier ? d->group_id[i] : 0]++;
  std::vector<int> bucket_ptr, bucket_rows;
  if (!m.hv) {
    bucket_ptr.assign(m.K + 1, 0);
    bucket_rows.resize(n);
    for (int64_t i = 0; i < n; ++i) ++bucket_ptr[f->test_index[i] + 1];
    for (int k = 0; k < m.K; ++k) bucket_ptr[k + 1] += bucket_ptr[k];
    std::vector<int> fill(bucket_ptr.begin(), bucket_ptr.end() - 1);
    for (int64_t i = 0; i < n; ++i) bucket_rows[fill[f->test_index[i]]++] = static_cast<int>(i);
  }
  std::vector<int> seg_group, seg_unseen, seg_rows;
  m.fold_seg.assign(m.K + 2, 0);
  m.seg_row.assign(1, 0);
  std::vector<int64_t> excl(Jg, 0), cnt(Jg, 0), start(Jg, 0);
  std::vector<int> tmp, order_rows;
  for (int k = 0; k < m.K; ++k) {
    m.fold_seg[k] = static_cast<int>(seg_group.size());
    tmp.clear();
    if (!m.hv) {
      for (int t = bucket_ptr[k]; t < bucket_ptr[k + 1]; ++t) tmp.push_back(bucket_rows[t]);
    } else {
      for (int64_t i = 0; i < n; ++i)
        if (rank[i] >= f->intervals[4 * k] && rank[i] < f->intervals[4 * k + 1]) tmp.push_back(static_cast<int>(i));
    }
    std::fill(excl.begin(), excl.end(), 0);
    std::fill(cnt.begin(), cnt.end(), 0);
    if (!m.hv) {
      for (int i : tmp) excl[hier ? d->group_id[i] : 0]++;
    } else if (hier) {
      for (int64_t i = 0; i < n; ++i)
        if (rank[i] >= f->intervals[4 * k + 2] && rank[i] < f->intervals[4 * k + 3]) excl[d->group_id[i]]++;
    }
    for (int i : tmp) cnt[hier ? d->group_id[i] : 0]++;
    int64_t acc = 0;
    for (int g = 0; g < Jg; ++g) {
      start[g] = acc;
      acc += cnt[g];
    }
    order_rows.assign(tmp.size(), 0);
    for (int i : tmp) order_rows[start[hier ? d->group_id[i] : 0]++] = i;
    size_t off = 0;
    for (int g = 0; g < Jg; ++g) {
      if (cnt[g] == 0) continue;
      seg_group.push_back(hier ? g : -1);
      seg_unseen.push_back(hier ? (gsize[g] - excl[g] == 0 ? 1 : 0) : 0);
      for (int64_t t = 0; t < cnt[g]; ++t) seg_rows.push_back(inv[order_rows[off + t]]);
      off += cnt[g];
      m.seg_row.push_back(static_cast<int>(seg_rows.size()));
    }
  }
  m.seg_rows = seg_rows;
  m.y_host.assign(y.begin(), y.begin() + n);
  m.fold_seg[m.K] = static_cast<int>(seg_group.size());
  m.fold_seg[m.K + 1] = static_cast<int>(seg_group.size());
  m.fseg.upload(m.fold_seg);
  m.sgroup.upload(seg_group.empty() ? std::vector<int>{0} : seg_group);
  m.sunseen.upload(seg_unseen.empty() ? std::vector<int>{0} : seg_unseen);
  m.srow.upload(m.seg_row);
  m.srows.upload(seg_rows.empty() ? std::vector<int>{0} : seg_rows);

  m.inv_mass.upload(std::vector<double>(kp->inv_mass_diag, kp->inv_mass_diag + m.dim));
  m.bank.upload(std::vector<double>(bank, bank + bank_rows * m.dim));
  m.bank_rows = bank_rows;

  ModelDev& md = m.md;
  md.family = s->family == PCVG_FAMILY_RAT_GROWTH ? (s->per_subject_slope ? kRatA : kRatB) : s->family;
  md.goff = m.dim - m.ng;
  md.n = static_cast<int>(n);
  md.nc = m.nc;
  md.J = m.J;
  md.ng = m.ng;
  md.dim = m.dim;
  md.K = m.K;
  md.broken_fold = -1;
  md.glm_part = nullptr;
  md.glm_cnt = nullptr;
  md.y = m.y.p;
  md.x = m.x.p;
  md.xr = m.xr.p;
  md.nc_pad = nc_pad;
  md.key = m.key.p;
  md.grp_ptr = m.grp_ptr.p;
  md.fold_lo = m.lo.p;
  md.fold_hi = m.hi.p;
  md.n_train = m.ntrain.p;
  md.fold_seg = m.fseg.p;
  md.seg_group = m.sgroup.p;
  md.seg_unseen = m.sunseen.p;
  md.any_unseen = std::any_of(seg_unseen.begin(), seg_unseen.end(), [](int u) { return u != 0; }) ? 1 : 0;
  md.seg_row = m.srow.p;
  md.seg_rows = m.srows.p;
  md.inv_mass = m.inv_mass.p;
  md.step = kp->step_size;
  md.n_lf = kp->n_leapfrog;
  for (int c = 0; c < kMaxCov; ++c)
    md.cmask[c] = (s->family == PCVG_FAMILY_GROUPED && c < m.nc)
                      ? ((s->covariate_mask == nullptr || s->covariate_mask[c]) ? 1.0 : 0.0)
                      : 0.0;
  md.include_floor = s->include_floor != 0;
  md.p = s->ar_order;
  md.q = s->dummies;
  md.rho_sym = s->rho_transform == PCVG_RHO_SYMMETRIC;
  // prior normalising constants with glibc (priors.hpp:13-26)
  md.c_lhn10 = 0.5 * std::log(2.0 / (3.141592653589793238462643383279 * 10.0));
  md.c_lhn1 = 0.5 * std::log(2.0 / (3.141592653589793238462643383279 * 1.0));
  md.c_lgamma6_9 = 6.0 * std::log(9.0) - std::lgamma(6.0);
  md.c_lgamma10_10 = 10.0 * std::log(10.0) - std::lgamma(10.0);
  md.c_lbeta55 = std::lgamma(10.0) - std::lgamma(5.0) - std::lgamma(5.0);
  md.c_log4 = std::log(4.0);
  md.c_lg25_2 = 25.0 * std::log(2.0) - std::lgamma(25.0);
  md.c_lg5_10 = 5.0 * std::log(10.0) - std::lgamma(5.0);
  md.c_lg1_2 = 1.0 * std::log(2.0) - std::lgamma(1.0);
  md.c_log20 = std::log(20.0);
  md.c_log2 = std::log(2.0);
  if (md.family == kRatA)  // the dense unseen-subject predictive runs in registers
    for (size_t sg = 0; sg < seg_unseen.size(); ++sg)
      if (seg_unseen[sg] && m.seg_row[sg + 1] - m.seg_row[sg] > 16)
        throw Error(PCVG_INVALID_INPUT, "per-subject growth model supports at most 16 observations per unseen subject on device");
  md.nb = nb;
  md.bstride = bstride;
  md.bgroup = m.bgroup.p;
  md.boff = m.boff.p;
  md.yb = m.yb.p;
  md.xb = m.xb.p;
  md.keyb = m.keyb.p;
  md.ntile = ntile;
  md.rt = rt;
  md.tile_first = m.tfirst.p;
  md.tile_r0 = m.tr0.p;
  md.tile_rows = m.trows.p;
  md.bkey_uniform = bkey_uniform;
  md.bkey = m.bkey.p;
  md.bgrows = m.bgrows.p;
  md.buniform = m.buni.p;
  md.ring = ring;
  md.x32 = m.x32.p;
  md.suff = suff;
  for (int i = 0; i <= kMaxCov; ++i) md.su[i] = suff && i < static_cast<int>(ss.ubar.size()) ? ss.ubar[i] : 0.0;
  md.sd = ss.d;
  md.sdp = ss.dp;
  md.sA = m.sA.p;
  md.sgn = m.sgn.p;
  md.sgs = m.sgs.p;
  md.sov_ptr = m.sov_ptr.p;
  md.sov_g = m.sov_g.p;
  md.sov_n = m.sov_n.p;
  md.sov_s = m.sov_s.p;
  md.sex_lo = m.sex_lo.p;
  md.sex_hi = m.sex_hi.p;
  md.sex_rows = m.sex_rows.p;
  md.sex_grp = m.sex_grp.p;
  md.sgA = m.sgA.p;
  md.sov_A = m.sov_A.p;
  return hm;
}

// Tensor-core GLM kernel or the generic lane-split kernel: the GLM path needs a
// predictor without group effects; for few chains it only pays once a cluster split fills the GPU.
bool use_glm(const pcvg_ctx* ctx, const HostModel& m, int nch) {
  if (m.md.nc_pad == 0) return false;
  if (m.family == PCVG_FAMILY_LOGISTIC) return true;  // no generic kernel for the logit link
  if (ctx->policy == PCVG_KERNEL_GENERIC) return false;
  if (ctx->policy == PCVG_KERNEL_TENSOR) return true;
  const int tiles = (nch + 63) / 64;
  return tiles * glm_cluster_size(m.md.n, m.md.nc_pad, nch) >= 24;
}

// md_override: the model with a different kernel (step size, n_leapfrog, inverse mass) - used by
// the full-data adaptation, whose kernel changes between transitions.
void launch_family(pcvg_ctx* ctx, const HostModel& m, const ChainsDev& S, const RunArgs& A,
                   cudaStream_t st = nullptr, const ModelDev* md_override = nullptr) {
  if (!st) st = ctx->stream;
  const ModelDev& md = md_override ? *md_override : m.md;
  const int launches0 = sampler_launch_count();
  cudaError_t e;
  if (ctx->policy == PCVG_KERNEL_TF32 && md.family == kLogistic && md.x32) {
    const size_t need = glm32_scratch_doubles(S.nch);
    if (m.g32.n < need) m.g32.alloc(need);
    ModelDev md32 = md;
    md32.g32_scratch = m.g32.p;
    e = launch_glm32(md32, S, A, st);  // FP32 variant: tcgen05 kind::tf32, split operands
  } else if ((ctx->policy == PCVG_KERNEL_SUFFSTAT || ctx->policy == PCVG_KERNEL_AUTO) && md.suff) {
    // fold sufficient statistics: the lean all-global kernel for warm-up / sampling where it applies
    static const bool no_lean = std::getenv("PCVG_NO_LEAN") != nullptr;  // A/B tests only
    const int T = suff_lanes_per_chain(md, S.nch);
    e = cudaErrorNotSupported;
    if (T == 1 && !no_lean) e = launch_lean(md, S, A, st);
    if (e == cudaErrorNotSupported) {
      cudaGetLastError();
      e = launch_gauss(md, S, A, -T, st);
    }
  } else if (use_glm(ctx, m, S.nch)) {
    ModelDev mdg = md;
    if ((S.nch + 63) / 64 <= 8) {
      // few chain tiles: the launcher may split each tile over several clusters (a cooperative
      // launch with a second reduction level in global memory); it runs on the context's first
      // stream, ordered with the other model's launches
      size_t pd = 0, nct = 0;
      glm_multicluster_scratch(md.nc_pad, S.nch, &pd, &nct);
      if (m.glm_part.n < pd) m.glm_part.alloc(pd);
      if (m.glm_cnt.n < nct) m.glm_cnt.alloc(nct);
      mdg.glm_part = m.glm_part.p;
      mdg.glm_cnt = m.glm_cnt.p;
      st = ctx->stream;
    }
    e = launch_glm(mdg, S, A, st);
  } else if (md.nb > 0 && (ctx->policy != PCVG_KERNEL_GENERIC || md.family >= kRatB)) {
    e = launch_gauss(md, S, A, 0, st);  // group-batched hierarchical kernel
  } else {
    const int T = gauss_lanes_per_chain(md, S.nch);
    e = launch_gauss(md, S, A, T, st);
  }
  ctx->launches += sampler_launch_count() - launches0;  // two when a wave tail is split
  ck(e, "kernel launch");
}

RunArgs make_args(int mode, int64_t n_iters) {
  RunArgs a{};
  a.mode = mode;
  a.n_iters = n_iters;
  return a;
}

int effective_batch(const pcvg_run_config* c) {  // engine.cpp:5-9
  if (c->batch_size > 0) return c->batch_size;
  return std::max(1, static_cast<int>(std::sqrt(static_cast<double>(c->iters) * c->chains)));
}

// Shuffle sub-blocks stored per chain: RunConfig::blocks, or one per check interval under early
// stop (regrouped into `blocks` benchmark blocks at each checkpoint).
int sub_block_count(const pcvg_run_config* c) {
  return c->early_stop ? static_cast<int>(c->iters / c->checkpoint_every) : c->blocks;
}

// Sub-blocks completed after iter_count sampling iterations (a checkpoint).
int completed_sub_blocks(const pcvg_run_config* c, int64_t iter_count) {
  if (!c->early_stop) return c->blocks;
  return static_cast<int>(std::clamp<int64_t>(iter_count / c->checkpoint_every, 1, c->iters / c->checkpoint_every));
}

void validate_run(const pcvg_ctx* ctx, const pcvg_run_config* c) {
  if (!c) throw Error(PCVG_INVALID_INPUT, "null run config");
  // RunConfig::validate, engine.cpp:21-30
  if (c->chains < 2) throw Error(PCVG_INVALID_INPUT, "need at least 2 chains per fold (Rhat)");
  if (c->iters < 1) throw Error(PCVG_INVALID_INPUT, "need at least 1 sampling iteration");
  if (c->warmup < 0) throw Error(PCVG_INVALID_INPUT, "warmup must be non-negative");
  if (c->iters < effective_batch(c)) throw Error(PCVG_INVALID_INPUT, "chain length must cover at least one batch");
  if (c->blocks < 1) throw Error(PCVG_INVALID_INPUT, "need at least 1 shuffle block");
  if (c->bench_draws < 1) throw Error(PCVG_INVALID_INPUT, "need at least 1 benchmark draw");
  if (c->checkpoint_every < 0) throw Error(PCVG_INVALID_INPUT, "checkpoint_every must be >= 0");
  if (c->chains > 64) throw Error(PCVG_INVALID_INPUT, "at most 64 chains per fold on device");
  // run_pcv preconditions, engine.cpp:258-271
  if (ctx->models.empty() || ctx->models.size() > 2)
    throw Error(PCVG_INVALID_INPUT, "run_pcv takes one or two models");
  const int K = ctx->models[0]->K;
  for (const auto& m : ctx->models)
    if (m->K != K) throw Error(PCVG_INVALID_INPUT, "models must share one fold assignment");
  if (c->score != PCVG_SCORE_LOGS && c->score != PCVG_SCORE_HS && c->score != PCVG_SCORE_DSS)
    throw Error(PCVG_INVALID_INPUT, "unknown score");
  // Model::check_score_support (model.cpp:21-28): the Gaussian families implement pred_derivs /
  // pred_sample; the logistic family (binary outcome) implements neither.
  for (const auto& m : ctx->models)
    if (c->score != PCVG_SCORE_LOGS && m->family == PCVG_FAMILY_LOGISTIC)
      throw Error(PCVG_UNSUPPORTED_SCORE, std::string("model does not support score ") +
                                              (c->score == PCVG_SCORE_HS ? "hs" : "dss"));
  if (K < 2) throw Error(PCVG_INVALID_INPUT, "uncertainty estimates need at least 2 folds");
  if (c->fold_begin < 0 || c->fold_end < c->fold_begin || c->fold_end > K)
    throw Error(PCVG_INVALID_INPUT, "bad fold shard");
  if (c->early_stop) {
    if (c->checkpoint_every <= 0 || c->iters % c->checkpoint_every != 0)
      throw Error(PCVG_INVALID_INPUT, "early_stop needs checkpoint_every dividing iters");
    // the rule needs at least `blocks` completed check intervals to form the benchmark's blocks
    if (c->iters / c->checkpoint_every < c->blocks)
      throw Error(PCVG_INVALID_INPUT, "early_stop needs iters / checkpoint_every >= blocks");
  }
}

int test_size_of(const HostModel& m, int fold) {
  return fold >= m.K ? 0 : m.seg_row[m.fold_seg[fold + 1]] - m.seg_row[m.fold_seg[fold]];
}

// HS / DSS state of a shard (ExtraDev layout, types.cuh): per local fold the test size, the
// accumulator / warm-up / centre bases; accumulators and warm-up sums start at zero.
void alloc_extra(ChainSet& cs, const HostModel& m, int kind, int fb, int nfold, int L) {
  cs.xkind = kind;
  cs.xm.resize(nfold);
  cs.xbase_h.resize(nfold);
  cs.xwbase_h.resize(nfold);
  cs.xcbase_h.resize(nfold);
  int64_t ab = 0, wb = 0, cb = 0;
  for (int k = 0; k < nfold; ++k) {
    const int mk = test_size_of(m, fb + k);
    cs.xm[k] = mk;
    cs.xbase_h[k] = ab;
    cs.xwbase_h[k] = wb;
    cs.xcbase_h[k] = cb;
    ab += L * extra_acc_len(kind, mk);
    wb += L * extra_warm_len(kind, mk);
    cb += extra_warm_len(kind, mk);
  }
  cs.xmsize.upload(cs.xm);
  cs.xbase.upload(cs.xbase_h);
  cs.xwbase.upload(cs.xwbase_h);
  cs.xcbase.upload(cs.xcbase_h);
  cs.xacc.alloc(std::max<int64_t>(ab, 1));
  cs.xwarm.alloc(std::max<int64_t>(wb, 1));
  cs.xdev.alloc(std::max<int64_t>(wb, 1));
  cs.xcenter.alloc(std::max<int64_t>(cb, 1));
  dzero(cs.xacc.p, sizeof(double) * cs.xacc.n);
  dzero(cs.xwarm.p, sizeof(double) * cs.xwarm.n);
}

// Per-fold HS / DSS estimates of a shard at `iters` sampling iterations (engine.cpp:148-171):
// chain merge on device, scores on the host. Overwrites estimate, ORs DSS failures into fault.
void extra_estimates(pcvg_ctx* ctx, const HostModel& m, const ChainSet& cs, int fb, int nfold,
                     int L, int64_t iters, double* estimate, int32_t* fault, int32_t* ridged) {
  const ChainsDev S = cs.view(L, fb, 0, 0);
  DevBuf<double> merged;
  merged.alloc(std::max<int64_t>(cs.xacc.n / L, 1));
  ck(launch_extra_merge(S, nfold, merged.p, ctx->stream), "extra merge");
  ++ctx->launches;
  const auto mg = merged.download(ctx->stream);
  const auto cen = cs.xcenter.download(ctx->stream);
  const int64_t count = iters * L;
  std::vector<double> yt;
  for (int k = 0; k < nfold; ++k) {
    const int mk = cs.xm[k];
    const double* a = mg.data() + cs.xbase_h[k] / L;
    const double* c = cen.data() + cs.xcbase_h[k];
    int rg = 0;
    if (cs.xkind == PCVG_SCORE_HS) {
      estimate[k] = hs_fold_estimate(a, c, mk, count);
    } else {
      const int fold = fb + k;
      yt.clear();  // Model::test_values (fold_meta order)
      for (int t = m.seg_row[m.fold_seg[fold]]; t < m.seg_row[m.fold_seg[fold + 1]]; ++t)
        yt.push_back(m.y_host[m.seg_rows[t]]);
      double sc;
      if (dss_fold_estimate(a, c, yt.data(), mk, count, &sc, &rg)) {
        estimate[k] = sc;
      } else {
        estimate[k] = std::numeric_limits<double>::quiet_NaN();
        fault[k] = 1;
      }
    }
    if (ridged) ridged[k] = rg;
  }
}

// Shuffle benchmark of the shard on device (bench_kernel): replicate maxima + rejection flags.
void device_benchmark(pcvg_ctx* ctx, const int32_t* failed, int64_t nonfailed_before,
                      int64_t nonfailed_total, int sub_used, double* rep_max, int32_t* needs_host) {
  const pcvg_run_config& cfg = ctx->cfg;
  const int nfold = ctx->fe - ctx->fb, L = cfg.chains, R = cfg.bench_draws;
  DevBuf<unsigned long long> mx;
  DevBuf<int> rj;
  mx.alloc(std::max(R, 1));
  rj.alloc(std::max(R, 1));
  ck(cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long) * mx.n, ctx->stream), "memset");
  ck(cudaMemsetAsync(rj.p, 0, sizeof(int) * rj.n, ctx->stream), "memset");
  for (size_t mi = 0; mi < ctx->chains.size(); ++mi) {  // one chain set per model (or score-stream run)
    std::vector<int64_t> item(nfold, -1);
    int64_t j = 0;
    for (int k = 0; k < nfold; ++k)
      if (!(failed && failed[k])) item[k] = static_cast<int64_t>(mi) * nonfailed_total + nonfailed_before + j++;
    DevBuf<int64_t> it;
    it.upload(item);
    const ChainSet& cs = *ctx->chains[mi];
    ChainsDev S = cs.view(L, ctx->fb, cfg.seed, 0);
    const int groups = std::min(cfg.blocks, sub_used);
    DevBuf<double> gx, gx2;
    if (groups != sub_used) {  // early stop: regroup the completed check intervals once
      gx.alloc(static_cast<size_t>(groups) * cs.nch);
      gx2.alloc(static_cast<size_t>(groups) * cs.nch);
      ck(launch_regroup(S, sub_used, groups, gx.p, gx2.p, ctx->stream), "regroup");
      ++ctx->launches;
      S.acc.y_x = gx.p;
      S.acc.y_x2 = gx2.p;
    }
    ck(launch_bench(S, nfold, it.p, R, groups, groups, ctx->iters_done, mx.p, rj.p, ctx->stream), "benchmark");
    ++ctx->launches;
    ck(cudaStreamSynchronize(ctx->stream), "benchmark");  // `it` is freed at scope exit
  }
  const auto m = mx.download(ctx->stream);
  const auto r = rj.download(ctx->stream);
  for (int i = 0; i < R; ++i) {
    double v;
    std::memcpy(&v, &m[i], sizeof v);
    rep_max[i] = v;
    needs_host[i] = r[i];
  }
}

void require_device(pcvg_ctx* ctx) {
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
}

}  // namespace

extern "C" {

int32_t pcvg_abi_version(void) { return PCVG_ABI_VERSION; }

const char* pcvg_last_error(const pcvg_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

const char* pcvg_status_name(int32_t s) {
  switch (s) {
    case PCVG_OK: return "ok";
    case PCVG_INVALID_INPUT: return "invalid_input";
    case PCVG_NUMERIC_FAULT: return "numeric_fault";
    case PCVG_ADAPTATION_FAILURE: return "adaptation_failure";
    case PCVG_UNDEFINED_DIAGNOSTIC: return "undefined_diagnostic";
    case PCVG_UNSUPPORTED_SCORE: return "unsupported_score";
    case PCVG_CUDA_ERROR: return "cuda_error";
    case PCVG_COMM_ERROR: return "comm_error";
  }
  return "unknown";
}

pcvg_status pcvg_rng_sequence(uint64_t seed, uint64_t stream, int32_t do_skip, uint64_t skip_block,
                              const char* ops, const uint64_t* arg, int64_t n, double* out) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { rng_sequence(seed, stream, do_skip, skip_block, ops, arg, n, out); }));
}
pcvg_status pcvg_make_loo(int64_t n, int32_t* ti, int32_t* K) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { make_loo(n, ti, K); }));
}
pcvg_status pcvg_make_logo(const pcvg_dataset* d, int32_t* ti, int32_t* K) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { make_logo(d, ti, K); }));
}
pcvg_status pcvg_make_kfold(int64_t n, int32_t K, uint64_t seed, int32_t* ti) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { make_kfold(n, K, seed, ti); }));
}
pcvg_status pcvg_make_time_blocks(const pcvg_dataset* d, int32_t K, int32_t* ti) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { make_time_blocks(d, K, ti); }));
}
pcvg_status pcvg_make_hv_block(const pcvg_dataset* d, int32_t K, int64_t h, int64_t* iv) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { make_hv_block(d, K, h, iv); }));
}
pcvg_status pcvg_make_hv_racine(const pcvg_dataset* d, int64_t v, int64_t h, int64_t* iv) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { make_hv_racine(d, v, h, iv); }));
}
pcvg_status pcvg_simulate_grouped(int32_t J, int32_t Nj, int32_t P, double mb, uint64_t seed,
                                  double* y, double* x, int32_t* g) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { simulate_grouped(J, Nj, P, mb, seed, y, x, g); }));
}
pcvg_status pcvg_simulate_radon(int32_t houses, int32_t counties, uint64_t seed, double* y,
                                double* x, int32_t* g) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { simulate_radon(houses, counties, seed, y, x, g); }));
}
pcvg_status pcvg_simulate_rat(int32_t subjects, uint64_t seed, double* y, double* x, int32_t* g) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { simulate_rat(subjects, seed, y, x, g); }));
}
pcvg_status pcvg_simulate_seasonal(int64_t months, int32_t p, int32_t q, double rho, double amp,
                                   double sigma, uint64_t seed, double* y, double* x, int64_t* t) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { simulate_seasonal(months, p, q, rho, amp, sigma, seed, y, x, t); }));
}
pcvg_status pcvg_simulate_linreg(int64_t n, int32_t P, uint64_t seed, double* y, double* x, int32_t* g) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { simulate_linreg(n, P, seed, y, x, g); }));
}
pcvg_status pcvg_simulate_logistic(int64_t n, int32_t P, uint64_t seed, double* y, double* x) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] { simulate_logistic(n, P, seed, y, x); }));
}

pcvg_status pcvg_create(int32_t device, pcvg_ctx** out) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] {
    if (!out) throw Error(PCVG_INVALID_INPUT, "null output");
    int count = 0;
    ck(cudaGetDeviceCount(&count), "no CUDA device (the PCV sampler has no CPU fallback)");
    if (device < 0 || device >= count) throw Error(PCVG_CUDA_ERROR, "device index out of range");
    auto ctx = std::make_unique<pcvg_ctx>();
    ctx->device = device;
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&ctx->evj, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreate(&ctx->ev0), "cudaEventCreate");
    ck(cudaEventCreate(&ctx->ev1), "cudaEventCreate");
    retain_pool_memory();
    *out = ctx.release();
  }));
}

pcvg_status pcvg_destroy(pcvg_ctx* ctx) {
  if (!ctx) return PCVG_OK;
  cudaSetDevice(ctx->device);
  static const bool verbose = std::getenv("PCVG_VERBOSE") != nullptr;  // tuning only
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t0 = now();
  cudaDeviceSynchronize();
  const auto t1 = now();
  ctx->chains.clear();
  const auto t2 = now();
  ctx->centers.clear();
  ctx->models.clear();
  ctx->stream_scores.alloc(0);  // every device buffer is freed in its stream's order before the streams go
  const auto t3 = now();
  if (verbose)
    std::fprintf(stderr, "pcvg_destroy: sync %.3f s, chains %.3f s, models %.3f s\n",
                 std::chrono::duration<double>(t1 - t0).count(), std::chrono::duration<double>(t2 - t1).count(),
                 std::chrono::duration<double>(t3 - t2).count());
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->evj) cudaEventDestroy(ctx->evj);
  if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return PCVG_OK;
}

pcvg_status pcvg_add_model(pcvg_ctx* ctx, const pcvg_dataset* data, const pcvg_folds* folds,
                           const pcvg_model_spec* spec, const pcvg_kernel* kernel,
                           const double* bank, int64_t bank_rows, int32_t model_id, int32_t* slot) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx) throw Error(PCVG_INVALID_INPUT, "null context");
    if (ctx->models.size() >= 2) throw Error(PCVG_INVALID_INPUT, "run_pcv takes one or two models");
    require_device(ctx);
    ctx->models.push_back(build_model(data, folds, spec, kernel, bank, bank_rows, model_id));
    ctx->begun = false;
    if (slot) *slot = static_cast<int32_t>(ctx->models.size() - 1);
  }));
}

pcvg_status pcvg_debug_break_fold(pcvg_ctx* ctx, int32_t slot, int32_t fold) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || slot < 0 || slot >= static_cast<int>(ctx->models.size())) throw Error(PCVG_INVALID_INPUT, "bad slot");
    if (fold < -1 || fold >= ctx->models[slot]->K) throw Error(PCVG_INVALID_INPUT, "fold out of range");
    ctx->models[slot]->md.broken_fold = fold;
  }));
}

pcvg_status pcvg_set_kernel_policy(pcvg_ctx* ctx, int32_t policy) {
  if (!ctx || policy < PCVG_KERNEL_AUTO || policy > PCVG_KERNEL_ROWS) return PCVG_INVALID_INPUT;
  ctx->policy = policy;
  return PCVG_OK;
}

pcvg_status pcvg_model_dim(const pcvg_ctx* ctx, int32_t slot, int32_t* dim) {
  if (!ctx || slot < 0 || slot >= static_cast<int>(ctx->models.size()) || !dim) return PCVG_INVALID_INPUT;
  *dim = ctx->models[slot]->dim;
  return PCVG_OK;
}

pcvg_status pcvg_model_test_size(const pcvg_ctx* ctx, int32_t slot, int32_t fold, int64_t* n) {
  if (!ctx || slot < 0 || slot >= static_cast<int>(ctx->models.size()) || !n) return PCVG_INVALID_INPUT;
  const HostModel& m = *ctx->models[slot];
  if (fold < 0 || fold > m.K) return PCVG_INVALID_INPUT;
  *n = fold == m.K ? 0 : m.seg_row[m.fold_seg[fold + 1]] - m.seg_row[m.fold_seg[fold]];
  return PCVG_OK;
}

}  // extern "C"

namespace {

// Temporary chain set for the parity probes: n chains at explicit (fold, theta).
std::unique_ptr<ChainSet> probe_chains(pcvg_ctx* ctx, const HostModel& m, int64_t n,
                                       const int32_t* fold, const double* theta) {
  for (int64_t i = 0; i < n; ++i)
    if (fold[i] < 0 || fold[i] > m.K) throw Error(PCVG_INVALID_INPUT, "fold id out of range (0..K)");
  auto cs = std::make_unique<ChainSet>();
  cs->alloc(static_cast<int>(n), m.dim, 1);
  std::vector<double> pos(2 * static_cast<size_t>(m.dim) * n, 0.0);
  for (int64_t c = 0; c < n; ++c)
    for (int d = 0; d < m.dim; ++d) pos[static_cast<size_t>(d) * n + c] = theta[c * m.dim + d];
  h2d(cs->pos.p, pos.data(), sizeof(double) * pos.size());
  dzero(cs->grad.p, sizeof(double) * cs->grad.n);
  dzero(cs->cur.p, n);
  dzero(cs->rpos.p, sizeof(uint64_t) * n);
  dzero(cs->has.p, n);
  dzero(cs->cached.p, sizeof(double) * n);
  dzero(cs->div.p, sizeof(int64_t) * n);
  dzero(cs->warm.p, sizeof(double) * n);
  dzero(cs->stream.p, sizeof(uint64_t) * n);
  cs->fold_override.upload(std::vector<int>(fold, fold + n));
  (void)ctx;
  return cs;
}

}  // namespace

extern "C" {

pcvg_status pcvg_eval(pcvg_ctx* ctx, int32_t slot, int64_t n, const int32_t* fold,
                      const double* theta, double* log_joint, double* grad) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || slot < 0 || slot >= static_cast<int>(ctx->models.size())) throw Error(PCVG_INVALID_INPUT, "bad slot");
    require_device(ctx);
    const HostModel& m = *ctx->models[slot];
    if (n < 1) return;
    auto cs = probe_chains(ctx, m, n, fold, theta);
    DevBuf<double> out;
    out.alloc(n);
    RunArgs a = make_args(kModeEval, 0);
    a.out_a = out.p;
    launch_family(ctx, m, cs->view(1, 0, 0, 0), a);
    ck(cudaStreamSynchronize(ctx->stream), "eval");
    const auto lj = out.download(ctx->stream);
    const auto g = cs->grad.download(ctx->stream);
    for (int64_t c = 0; c < n; ++c) {
      if (log_joint) log_joint[c] = lj[c];
      if (grad)
        for (int d = 0; d < m.dim; ++d) grad[c * m.dim + d] = g[static_cast<size_t>(d) * n + c];
    }
  }));
}

pcvg_status pcvg_eval_pred(pcvg_ctx* ctx, int32_t slot, int64_t n, const int32_t* fold,
                           const double* theta, double* log_pred) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || slot < 0 || slot >= static_cast<int>(ctx->models.size())) throw Error(PCVG_INVALID_INPUT, "bad slot");
    require_device(ctx);
    const HostModel& m = *ctx->models[slot];
    if (n < 1) return;
    auto cs = probe_chains(ctx, m, n, fold, theta);
    DevBuf<double> out;
    out.alloc(n);
    RunArgs a = make_args(kModePred, 1);
    a.out_a = out.p;
    launch_family(ctx, m, cs->view(1, 0, 0, 0), a);
    ck(cudaStreamSynchronize(ctx->stream), "eval_pred");
    const auto lp = out.download(ctx->stream);
    std::copy(lp.begin(), lp.end(), log_pred);
  }));
}

pcvg_status pcvg_hmc_probe(pcvg_ctx* ctx, int32_t slot, int64_t n, const int32_t* fold,
                           const double* theta, const double* momentum, const double* u,
                           double* theta_out, double* h0, double* h1, int32_t* accepted,
                           int32_t* divergent) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || slot < 0 || slot >= static_cast<int>(ctx->models.size())) throw Error(PCVG_INVALID_INPUT, "bad slot");
    require_device(ctx);
    const HostModel& m = *ctx->models[slot];
    if (n < 1) return;
    auto cs = probe_chains(ctx, m, n, fold, theta);
    const ChainsDev S = cs->view(1, 0, 0, 0);
    launch_family(ctx, m, S, make_args(kModeEval, 0));
    DevBuf<double> mom, uu, oa, ob;
    DevBuf<int32_t> fl;
    mom.upload(std::vector<double>(momentum, momentum + n * m.dim));
    uu.upload(std::vector<double>(u, u + n));
    oa.alloc(n);
    ob.alloc(n);
    fl.alloc(n);
    RunArgs a = make_args(kModeProbe, 1);
    a.probe_momentum = mom.p;
    a.probe_u = uu.p;
    a.out_a = oa.p;
    a.out_b = ob.p;
    a.out_flags = fl.p;
    launch_family(ctx, m, S, a);
    ck(cudaStreamSynchronize(ctx->stream), "hmc_probe");
    const auto a0 = oa.download(ctx->stream), b0 = ob.download(ctx->stream);
    const auto f0 = fl.download(ctx->stream);
    const auto pos = cs->pos.download(ctx->stream);
    const auto cur = cs->cur.download(ctx->stream);
    const size_t plane = static_cast<size_t>(m.dim) * n;
    for (int64_t c = 0; c < n; ++c) {
      if (h0) h0[c] = a0[c];
      if (h1) h1[c] = b0[c];
      if (accepted) accepted[c] = f0[c] & 1;
      if (divergent) divergent[c] = (f0[c] >> 1) & 1;
      for (int d = 0; d < m.dim; ++d) theta_out[c * m.dim + d] = pos[cur[c] * plane + static_cast<size_t>(d) * n + c];
    }
  }));
}

pcvg_status pcvg_leapfrog(pcvg_ctx* ctx, int32_t slot, int64_t n, const int32_t* fold,
                          const double* theta, const double* momentum, double* theta_out,
                          double* momentum_out, int32_t* ok) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || slot < 0 || slot >= static_cast<int>(ctx->models.size())) throw Error(PCVG_INVALID_INPUT, "bad slot");
    if (!theta || !momentum || !theta_out || !momentum_out) throw Error(PCVG_INVALID_INPUT, "null argument");
    require_device(ctx);
    const HostModel& m = *ctx->models[slot];
    if (n < 1) return;
    auto cs = probe_chains(ctx, m, n, fold, theta);
    DevBuf<double> pout;
    pout.alloc(static_cast<size_t>(n) * m.dim);
    ChainsDev S = cs->view(1, 0, 0, 0);
    S.probe_p_out = pout.p;
    launch_family(ctx, m, S, make_args(kModeEval, 0));
    DevBuf<double> mom, uu, oa, ob;
    DevBuf<int32_t> fl;
    mom.upload(std::vector<double>(momentum, momentum + n * m.dim));
    uu.upload(std::vector<double>(n, 0.0));  // log(0) < -dH: every finite trajectory is accepted
    oa.alloc(n);
    ob.alloc(n);
    fl.alloc(n);
    RunArgs a = make_args(kModeProbe, 1);
    a.probe_momentum = mom.p;
    a.probe_u = uu.p;
    a.out_a = oa.p;
    a.out_b = ob.p;
    a.out_flags = fl.p;
    a.traj = pout.p;
    launch_family(ctx, m, S, a);
    ck(cudaStreamSynchronize(ctx->stream), "leapfrog");
    const auto f0 = fl.download(ctx->stream);
    const auto pos = cs->pos.download(ctx->stream);
    const auto cur = cs->cur.download(ctx->stream);
    const auto po = pout.download(ctx->stream);
    const size_t plane = static_cast<size_t>(m.dim) * n;
    for (int64_t c = 0; c < n; ++c) {
      if (ok) ok[c] = (f0[c] >> 1) & 1 ? 0 : 1;
      for (int d = 0; d < m.dim; ++d) {
        theta_out[c * m.dim + d] = pos[cur[c] * plane + static_cast<size_t>(d) * n + c];
        momentum_out[c * m.dim + d] = po[c * m.dim + d];
      }
    }
  }));
}

pcvg_status pcvg_hmc_chain(pcvg_ctx* ctx, int32_t slot, int32_t fold, int32_t chain, uint64_t seed,
                           const double* theta0, int64_t n_steps, double* trajectory,
                           int32_t* divergent) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || slot < 0 || slot >= static_cast<int>(ctx->models.size())) throw Error(PCVG_INVALID_INPUT, "bad slot");
    require_device(ctx);
    const HostModel& m = *ctx->models[slot];
    if (n_steps < 1) return;
    auto cs = probe_chains(ctx, m, 1, &fold, theta0);
    const uint64_t st = stream_key(PCVG_STREAM_CHAIN_SAMPLING, static_cast<uint64_t>(m.model_id),
                                   static_cast<uint64_t>(fold), static_cast<uint64_t>(chain));
    h2d(cs->stream.p, &st, sizeof st);
    ChainsDev S = cs->view(1, 0, seed, static_cast<uint64_t>(m.model_id));
    launch_family(ctx, m, S, make_args(kModeEval, 0));
    DevBuf<double> tr;
    DevBuf<int32_t> dv;
    tr.alloc(static_cast<size_t>(n_steps) * m.dim);
    dv.alloc(n_steps);
    RunArgs a = make_args(kModeChain, n_steps);
    a.traj = tr.p;
    a.traj_div = dv.p;
    launch_family(ctx, m, S, a);
    ck(cudaStreamSynchronize(ctx->stream), "hmc_chain");
    const auto t = tr.download(ctx->stream);
    const auto d = dv.download(ctx->stream);
    std::copy(t.begin(), t.end(), trajectory);
    if (divergent)
      for (size_t i = 0; i < d.size(); ++i) divergent[i] = (d[i] >> 1) & 1;
  }));
}

pcvg_status pcvg_score_streams(pcvg_ctx* ctx, int32_t L, int64_t n, const double* s, double center,
                               int32_t b, int32_t D, double* out) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || L < 1 || L > 64 || n < 1 || D < 1 || b < 1 || !s || !out)
      throw Error(PCVG_INVALID_INPUT, "bad stream probe");
    require_device(ctx);
    ChainSet cs;
    cs.alloc(L, 1, D);
    DevBuf<double> centers, streams;
    centers.upload(std::vector<double>{center});
    streams.upload(std::vector<double>(s, s + static_cast<size_t>(L) * n));
    ChainsDev S = cs.view(L, 0, 0, 0);
    dzero(cs.warm.p, sizeof(double) * L);
    ck(launch_centers(S, 0, 0, centers.p, D, ctx->stream), "reset");  // nfold 0: no centre recompute
    ck(launch_feed_streams(S, streams.p, n, 0, n, n, D, b, ctx->stream), "feed");
    DevBuf<double> o;
    o.alloc(6);
    DevBuf<int64_t> bt;
    bt.alloc(1);
    DevBuf<int32_t> ft;
    ft.alloc(1);
    ck(launch_fold_stats(S, 1, n, b, D, o.p, o.p + 1, o.p + 2, o.p + 3, o.p + 4, o.p + 5, bt.p, ft.p,
                         ctx->stream), "fold_stats");
    ctx->launches += 3;
    const auto v = o.download(ctx->stream);
    const auto bb = bt.download(ctx->stream);
    const auto ff = ft.download(ctx->stream);
    for (int i = 0; i < 6; ++i) out[i] = v[i];
    out[6] = static_cast<double>(bb[0]);
    out[7] = ff[0];
  }));
}

int32_t pcvg_checkpoint_count(const pcvg_run_config* cfg) {  // engine.cpp:279-283
  if (!cfg || cfg->iters < 1) return 0;
  int32_t n = 0;
  if (cfg->checkpoint_every > 0)
    for (int64_t t = cfg->checkpoint_every; t < cfg->iters; t += cfg->checkpoint_every) ++n;
  return n + 1;
}

pcvg_status pcvg_begin(pcvg_ctx* ctx, const pcvg_run_config* cfg) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx) throw Error(PCVG_INVALID_INPUT, "null context");
    validate_run(ctx, cfg);
    require_device(ctx);
    ctx->cfg = *cfg;
    ctx->b = effective_batch(cfg);
    const int K = ctx->models[0]->K;
    ctx->fb = cfg->fold_begin;
    ctx->fe = (cfg->fold_begin == 0 && cfg->fold_end == 0) ? K : cfg->fold_end;
    const int nfold = ctx->fe - ctx->fb;
    const int L = cfg->chains;
    const int D = sub_block_count(cfg);
    ctx->chains.clear();
    ctx->centers.clear();
    ctx->div_base.clear();
    ctx->stream_mode = false;
    ctx->stream_scores.alloc(0);
    ctx->iters_done = 0;
    ctx->sample_ms = 0.0;
    ck(cudaEventRecord(ctx->ev0, ctx->stream), "event");
    ck(cudaStreamWaitEvent(ctx->stream2, ctx->ev0, 0), "wait");
    for (size_t mi = 0; mi < ctx->models.size(); ++mi) {
      const HostModel& m = *ctx->models[mi];
      cudaStream_t st = mi == 0 ? ctx->stream : ctx->stream2;
      auto cs = std::make_unique<ChainSet>();
      cs->alloc(nfold * L, m.dim, D);
      if (cfg->score != PCVG_SCORE_LOGS) alloc_extra(*cs, m, cfg->score, ctx->fb, nfold, L);
      const uint64_t sm = cfg->shared_streams ? 0u : static_cast<uint64_t>(m.model_id);
      const ChainsDev S = cs->view(L, ctx->fb, cfg->seed, sm);
      ck(launch_init_chains(m.md, S, m.bank.p, m.bank_rows, st), "init_chains");
      ++ctx->launches;
      launch_family(ctx, m, S, make_args(kModeEval, 0), st);
      if (cfg->warmup > 0) {
        RunArgs a = make_args(kModeWarmup, cfg->warmup);
        launch_family(ctx, m, S, a, st);
      }
      auto centers = std::make_unique<DevBuf<double>>();
      centers->alloc(std::max(nfold, 1));
      ck(launch_centers(S, nfold, cfg->warmup, centers->p, D, st), "centers");
      ctx->launches += 2;
      if (cfg->score != PCVG_SCORE_LOGS) {
        ck(launch_extra_centers(S, nfold, cfg->warmup, st), "extra centers");
        ++ctx->launches;
      }
      ctx->chains.push_back(std::move(cs));
      ctx->centers.push_back(std::move(centers));
    }
    ck(cudaEventRecord(ctx->evj, ctx->stream2), "event");
    ck(cudaStreamWaitEvent(ctx->stream, ctx->evj, 0), "wait");
    ck(cudaEventRecord(ctx->ev1, ctx->stream), "event");
    ck(cudaEventSynchronize(ctx->ev1), "warmup");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->warm_ms = ms;
    for (const auto& cs : ctx->chains) ctx->div_base.push_back(cs->div.download(ctx->stream));
    ctx->begun = true;
  }));
}

pcvg_status pcvg_advance(pcvg_ctx* ctx, int64_t n_iters) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || !ctx->begun) throw Error(PCVG_INVALID_INPUT, "pcvg_begin first");
    if (n_iters < 0 || ctx->iters_done + n_iters > ctx->cfg.iters)
      throw Error(PCVG_INVALID_INPUT, "advance past the planned chain length");
    require_device(ctx);
    const pcvg_run_config& cfg = ctx->cfg;
    ck(cudaEventRecord(ctx->ev0, ctx->stream), "event");
    ck(cudaStreamWaitEvent(ctx->stream2, ctx->ev0, 0), "wait");
    if (ctx->stream_mode && n_iters > 0) {
      const ChainSet& cs = *ctx->chains[0];
      ck(launch_feed_streams(cs.view(cfg.chains, 0, cfg.seed, 0), ctx->stream_scores.p, cfg.iters, ctx->iters_done,
                             ctx->iters_done + n_iters, cfg.iters, cs.D, ctx->b, ctx->stream), "feed");
      ++ctx->launches;
    }
    for (size_t mi = 0; mi < ctx->models.size() && !ctx->stream_mode; ++mi) {
      const HostModel& m = *ctx->models[mi];
      const uint64_t sm = cfg.shared_streams ? 0u : static_cast<uint64_t>(m.model_id);
      const ChainsDev S = ctx->chains[mi]->view(cfg.chains, ctx->fb, cfg.seed, sm);
      RunArgs a = make_args(kModeSample, n_iters);
      a.iter0 = ctx->iters_done;
      a.planned_n = cfg.iters;
      a.D = ctx->chains[mi]->D;
      a.b = ctx->b;
      if (n_iters > 0) launch_family(ctx, m, S, a, mi == 0 ? ctx->stream : ctx->stream2);
    }
    ck(cudaEventRecord(ctx->evj, ctx->stream2), "event");
    ck(cudaStreamWaitEvent(ctx->stream, ctx->evj, 0), "wait");
    ck(cudaEventRecord(ctx->ev1, ctx->stream), "event");
    ck(cudaEventSynchronize(ctx->ev1), "advance");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->last_ms = ms;
    ctx->sample_ms += ms;
    ctx->iters_done += n_iters;
  }));
}

pcvg_status pcvg_fold_stats(pcvg_ctx* ctx, pcvg_fold_table* out, int64_t* divergences,
                            int64_t* dropped, int64_t* iters_done) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || !ctx->begun) throw Error(PCVG_INVALID_INPUT, "pcvg_begin first");
    if (ctx->iters_done < 1) throw Error(PCVG_INVALID_INPUT, "no sampling iterations yet");
    require_device(ctx);
    const pcvg_run_config& cfg = ctx->cfg;
    const int nfold = ctx->fe - ctx->fb, L = cfg.chains;
    const int nm = static_cast<int>(ctx->chains.size());
    std::vector<std::vector<int64_t>> sdiv(nm);
    int64_t drop = 0;
    for (int mi = 0; mi < nm; ++mi) {
      const ChainSet& cs = *ctx->chains[mi];
      const ChainsDev S = cs.view(L, ctx->fb, cfg.seed, 0);
      DevBuf<double> est, lf, mc, nv, ess, rh;
      DevBuf<int64_t> bt;
      DevBuf<int32_t> ft;
      est.alloc(nfold); lf.alloc(nfold); mc.alloc(nfold); nv.alloc(nfold); ess.alloc(nfold); rh.alloc(nfold);
      bt.alloc(nfold); ft.alloc(nfold);
      ck(launch_fold_stats(S, nfold, ctx->iters_done, ctx->b, cs.D, est.p, lf.p, mc.p, nv.p, ess.p, rh.p, bt.p, ft.p, ctx->stream), "fold_stats");
      ++ctx->launches;
      const auto e = est.download(ctx->stream), l = lf.download(ctx->stream), c = mc.download(ctx->stream),
                 v = nv.download(ctx->stream), s = ess.download(ctx->stream), r = rh.download(ctx->stream);
      const auto b = bt.download(ctx->stream);
      const auto f = ft.download(ctx->stream);
      const size_t off = static_cast<size_t>(mi) * nfold;
      std::vector<double> ee = e;
      std::vector<int32_t> fx = f;
      std::vector<int32_t> rg(nfold, 0);
      if (cfg.score != PCVG_SCORE_LOGS)
        extra_estimates(ctx, *ctx->models[mi], cs, ctx->fb, nfold, L, ctx->iters_done, ee.data(),
                        fx.data(), rg.data());
      for (int k = 0; k < nfold; ++k) {
        if (out->dss_ridged) out->dss_ridged[off + k] = rg[k];
        if (out->estimate) out->estimate[off + k] = ee[k];
        if (out->log_f_hat) out->log_f_hat[off + k] = l[k];
        if (out->mc_contribution) out->mc_contribution[off + k] = c[k];
        if (out->naive_contribution) out->naive_contribution[off + k] = v[k];
        if (out->ess) out->ess[off + k] = s[k];
        if (out->rhat) out->rhat[off + k] = r[k];
        if (out->batches) out->batches[off + k] = b[k];
        if (out->fault) out->fault[off + k] = fx[k];
      }
      const auto dv = cs.div.download(ctx->stream);
      sdiv[mi].resize(dv.size());
      for (size_t i = 0; i < dv.size(); ++i) sdiv[mi][i] = dv[i] - ctx->div_base[mi][i];
      if (divergences)
        for (size_t i = 0; i < dv.size(); ++i) divergences[off * L + i] = sdiv[mi][i];
      const auto pend = cs.pending.download(ctx->stream);
      for (int32_t p : pend) drop += p;
    }
    // failed folds (engine.cpp:385-397): every chain of some model divergent on > N/2 iterations
    if (out->failed) {
      for (int k = 0; k < nfold; ++k) {
        bool failed = false;
        for (int mi = 0; mi < nm && !failed; ++mi) {
          bool all_bad = true;
          for (int c = 0; c < L; ++c)
            if (sdiv[mi][k * L + c] * 2 <= ctx->iters_done) { all_bad = false; break; }
          failed = all_bad;
        }
        for (int mi = 0; mi < nm; ++mi) out->failed[static_cast<size_t>(mi) * nfold + k] = failed ? 1 : 0;
      }
    }
    if (dropped) *dropped = drop;
    if (iters_done) *iters_done = ctx->iters_done;
  }));
}

pcvg_status pcvg_block_sums(pcvg_ctx* ctx, double* y_x, double* y_x2) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || !ctx->begun) throw Error(PCVG_INVALID_INPUT, "pcvg_begin first");
    require_device(ctx);
    size_t off = 0;
    for (const auto& cs : ctx->chains) {
      const auto a = cs->y_x.download(ctx->stream), b = cs->y_x2.download(ctx->stream);
      const int D = cs->D, n = cs->nch;
      for (int c = 0; c < n; ++c)
        for (int d = 0; d < D; ++d) {
          y_x[off + static_cast<size_t>(c) * D + d] = a[static_cast<size_t>(d) * n + c];
          y_x2[off + static_cast<size_t>(c) * D + d] = b[static_cast<size_t>(d) * n + c];
        }
      off += static_cast<size_t>(n) * D;
    }
  }));
}

pcvg_status pcvg_phase_times(const pcvg_ctx* ctx, double* warmup_ms, double* sampling_ms) {
  if (!ctx) return PCVG_INVALID_INPUT;
  if (warmup_ms) *warmup_ms = ctx->warm_ms;
  if (sampling_ms) *sampling_ms = ctx->sample_ms;
  return PCVG_OK;
}

pcvg_status pcvg_timing(const pcvg_ctx* ctx, double* last_ms, int64_t* launches) {
  if (!ctx) return PCVG_INVALID_INPUT;
  if (last_ms) *last_ms = ctx->last_ms;
  if (launches) *launches = ctx->launches;
  return PCVG_OK;
}

pcvg_status pcvg_merge(int32_t n_models, int32_t K, const pcvg_run_config* cfg, int64_t iter_count,
                       int32_t final_checkpoint, const pcvg_fold_table* folds, const double* y_x,
                       const double* y_x2, pcvg_report* report) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] {
    if (!cfg || !folds || !report || n_models < 1 || n_models > 2 || K < 2)
      throw Error(PCVG_INVALID_INPUT, "bad merge arguments");
    merge_stats(n_models, K, cfg, iter_count, final_checkpoint, folds, y_x, y_x2, completed_sub_blocks(cfg, iter_count),
                report, nullptr);
  }));
}

pcvg_status pcvg_benchmark(pcvg_ctx* ctx, const int32_t* failed, int64_t nonfailed_before,
                           int64_t nonfailed_total, int32_t blocks_used, double* rep_max,
                           int32_t* needs_host) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || !ctx->begun) throw Error(PCVG_INVALID_INPUT, "pcvg_begin first");
    if (ctx->iters_done < 1) throw Error(PCVG_INVALID_INPUT, "no sampling iterations yet");
    if (!rep_max || !needs_host || nonfailed_before < 0 || nonfailed_total < 0)
      throw Error(PCVG_INVALID_INPUT, "bad benchmark arguments");
    if (blocks_used < 1 || blocks_used > ctx->chains[0]->D) throw Error(PCVG_INVALID_INPUT, "blocks_used out of range");
    require_device(ctx);
    device_benchmark(ctx, failed, nonfailed_before, nonfailed_total, blocks_used, rep_max, needs_host);
  }));
}

pcvg_status pcvg_benchmark_host(int32_t n_models, int32_t nfold, int32_t L, int32_t D_stride,
                                int32_t blocks_used, int32_t block_groups, int64_t iter_count, uint64_t seed,
                                int32_t bench_draws, const double* y_x, const double* y_x2,
                                const int32_t* failed, int64_t nonfailed_before,
                                int64_t nonfailed_total, double* rep_max, int32_t* needs_host) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] {
    if (n_models < 1 || n_models > 2 || nfold < 0 || L < 2 || blocks_used < 1 || blocks_used > D_stride ||
        block_groups < 1 || block_groups > blocks_used || bench_draws < 0 || !y_x || !y_x2 || !rep_max || !needs_host)
      throw Error(PCVG_INVALID_INPUT, "bad benchmark arguments");
    bench_shard(n_models, nfold, L, D_stride, blocks_used, block_groups, iter_count, seed, bench_draws, y_x, y_x2,
                failed, nonfailed_before, nonfailed_total, rep_max, needs_host);
  }));
}

pcvg_status pcvg_merge_bench(int32_t n_models, int32_t K, const pcvg_run_config* cfg,
                             int64_t iter_count, int32_t final_checkpoint,
                             const pcvg_fold_table* folds, const double* bench_max,
                             pcvg_report* report) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] {
    if (!cfg || !folds || !report || !bench_max || n_models < 1 || n_models > 2 || K < 2)
      throw Error(PCVG_INVALID_INPUT, "bad merge arguments");
    merge_stats(n_models, K, cfg, iter_count, final_checkpoint, folds, nullptr, nullptr,
                completed_sub_blocks(cfg, iter_count), report, bench_max);
  }));
}

}  // extern "C"

namespace {

// Steps 3-4 of run_pcv (engine.cpp:342-483) on a begun context that owns every fold: advance to each
// checkpoint, per-fold statistics, snapshot merge; at the last checkpoint (or when the early-stop rule
// fires) the shuffle benchmark, exclusions and the final report.
void run_checkpoints(pcvg_ctx* ctx, const pcvg_run_config* cfg, pcvg_report* rep) {
  int32_t st = PCVG_OK;
  const int K = ctx->fe - ctx->fb, L = cfg->chains;
  const int nm = static_cast<int>(ctx->chains.size());
  const int D = ctx->chains[0]->D;
  std::vector<int64_t> cks;
  if (cfg->checkpoint_every > 0)
    for (int64_t t = cfg->checkpoint_every; t < cfg->iters; t += cfg->checkpoint_every) cks.push_back(t);
  cks.push_back(cfg->iters);
  // per-fold scratch table
  const size_t rows = static_cast<size_t>(nm) * K;
  std::vector<double> est(rows), lf(rows), mc(rows), nv(rows), ess(rows), rh(rows);
  std::vector<int64_t> bt(rows);
  std::vector<int32_t> ft(rows), fl(rows), rg(rows);
  pcvg_fold_table tab{est.data(), lf.data(), mc.data(), nv.data(), ess.data(), rh.data(), bt.data(), ft.data(), fl.data(), rg.data()};
  std::vector<double> yx(rows * L * D), yx2(rows * L * D);
  int64_t dropped = 0, done = 0;
  std::vector<int64_t> divs(rows * L);
  rep->n_checkpoints = 0;
  bool stopped = false;
  static const bool verbose = std::getenv("PCVG_VERBOSE") != nullptr;  // tuning only
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
  for (size_t ci = 0; ci < cks.size() && !stopped; ++ci) {
    const auto t0 = now();
    st = pcvg_advance(ctx, cks[ci] - ctx->iters_done);
    if (st != PCVG_OK) throw Error(st, ctx->err);
    const auto t1 = now();
    st = pcvg_fold_stats(ctx, &tab, divs.data(), &dropped, &done);
    if (st != PCVG_OK) throw Error(st, ctx->err);
    const auto t2 = now();
    const bool last = ci + 1 == cks.size();
    bool final_ck = last;
    if (cfg->early_stop && !last && static_cast<int>(ci + 1) >= cfg->blocks) {
      // Early-stop rule: the completed check intervals (sub-blocks) are regrouped into
      // `blocks` benchmark blocks, so the rule only looks once there are at least that many.
      pcvg_report probe = *rep;
      std::vector<double> bench(cfg->bench_draws);
      probe.benchmark = bench.data();
      probe.snapshots = nullptr;
      probe.delta_k = nullptr;
      pcvg_fold_table t2 = tab;
      t2.failed = nullptr;
      std::vector<double> bmax(cfg->bench_draws);
      std::vector<int32_t> bhost(cfg->bench_draws);
      device_benchmark(ctx, nullptr, 0, K, completed_sub_blocks(cfg, done), bmax.data(), bhost.data());
      const bool host_path = std::any_of(bhost.begin(), bhost.end(), [](int32_t v) { return v != 0; });
      if (host_path) {
        st = pcvg_block_sums(ctx, yx.data(), yx2.data());
        if (st != PCVG_OK) throw Error(st, ctx->err);
      }
      merge_stats(nm, K, cfg, done, 2, &t2, yx.data(), yx2.data(), completed_sub_blocks(cfg, done), &probe,
                  host_path ? nullptr : bmax.data());
      if (probe.verdict_pass && probe.benchmark_count > 0 && std::isfinite(probe.rhat_max) &&
          probe.mcse < probe.epistemic_se)
        final_ck = true;
    }
    if (final_ck) {
      // shuffle benchmark on device over the non-failed folds (failed flags from fold_stats)
      const int D_used = completed_sub_blocks(cfg, done);
      int64_t nonfailed = 0;
      for (int k = 0; k < K; ++k) nonfailed += fl[k] ? 0 : 1;
      std::vector<double> bmax(cfg->bench_draws);
      std::vector<int32_t> bhost(cfg->bench_draws);
      device_benchmark(ctx, fl.data(), 0, nonfailed, D_used, bmax.data(), bhost.data());
      const bool host_path = std::any_of(bhost.begin(), bhost.end(), [](int32_t v) { return v != 0; });
      if (host_path) {  // a below() rejection: the reference's sequential stream on the host
        st = pcvg_block_sums(ctx, yx.data(), yx2.data());
        if (st != PCVG_OK) throw Error(st, ctx->err);
      }
      merge_stats(nm, K, cfg, done, 1, &tab, yx.data(), yx2.data(), D_used, rep,
                  host_path ? nullptr : bmax.data());
      stopped = true;
    } else {
      pcvg_fold_table t2 = tab;
      t2.failed = nullptr;
      merge_stats(nm, K, cfg, done, 0, &t2, nullptr, nullptr, D, rep, nullptr);
    }
    if (verbose)
      std::fprintf(stderr, "checkpoint %zu (iteration %lld): advance %.3f s, fold_stats %.3f s, rule + merge %.3f s\n", ci,
                   static_cast<long long>(done), secs(t0, t1), secs(t1, t2), secs(t2, now()));
    if (rep->snapshots) {
      double* o = rep->snapshots + 7 * ci;
      o[0] = static_cast<double>(done);
      o[1] = rep->delta_hat;
      o[2] = rep->mcse;
      o[3] = rep->epistemic_se;
      o[4] = rep->prob_a_better;
      o[5] = rep->ess_overall;
      o[6] = rep->rhat_max;
    }
    rep->n_checkpoints = static_cast<int32_t>(ci + 1);
  }
  // final tables
  for (size_t i = 0; i < rows; ++i) {
    rep->folds.estimate[i] = est[i];
    rep->folds.log_f_hat[i] = lf[i];
    rep->folds.mc_contribution[i] = mc[i];
    if (rep->folds.naive_contribution) rep->folds.naive_contribution[i] = nv[i];
    rep->folds.ess[i] = ess[i];
    rep->folds.rhat[i] = rh[i];
    rep->folds.batches[i] = bt[i];
    rep->folds.fault[i] = ft[i];
    if (rep->folds.dss_ridged) rep->folds.dss_ridged[i] = rg[i];
  }
  // failed flags after exclusions are written by merge_stats into rep->folds.failed
  std::copy(divs.begin(), divs.end(), rep->divergences);
  rep->dropped_batch_draws = dropped;
  rep->iters_run = done;
  rep->warmup_ms = ctx->warm_ms;
  rep->sampling_ms = ctx->sample_ms;
  rep->gpu_launches = ctx->launches;
}

}  // namespace

extern "C" {

pcvg_status pcvg_run(pcvg_ctx* ctx, const pcvg_run_config* cfg, pcvg_report* rep) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || !rep) throw Error(PCVG_INVALID_INPUT, "null argument");
    if (cfg && (cfg->fold_begin != 0 || cfg->fold_end != 0) &&
        !(cfg->fold_begin == 0 && cfg->fold_end == (ctx->models.empty() ? 0 : ctx->models[0]->K)))
      throw Error(PCVG_INVALID_INPUT, "pcvg_run runs every fold; shard with the stepwise API");
    int32_t st = pcvg_begin(ctx, cfg);
    if (st != PCVG_OK) throw Error(st, ctx->err);
    run_checkpoints(ctx, cfg, rep);
  }));
}

pcvg_status pcvg_run_streams(pcvg_ctx* ctx, int32_t K, const double* s, const double* centers,
                             const pcvg_run_config* cfg, pcvg_report* rep) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || !s || !centers || !cfg || !rep) throw Error(PCVG_INVALID_INPUT, "null argument");
    if (!ctx->models.empty()) throw Error(PCVG_INVALID_INPUT, "score-stream runs need a context without models");
    const pcvg_run_config* c = cfg;
    if (c->chains < 2 || c->chains > 64) throw Error(PCVG_INVALID_INPUT, "need 2..64 chains per fold");
    if (c->iters < 1 || c->iters < effective_batch(c)) throw Error(PCVG_INVALID_INPUT, "chain length must cover a batch");
    if (c->blocks < 1 || c->bench_draws < 1 || c->checkpoint_every < 0 || K < 2)
      throw Error(PCVG_INVALID_INPUT, "bad run configuration");
    if (c->score != PCVG_SCORE_LOGS) throw Error(PCVG_UNSUPPORTED_SCORE, "score streams carry LogS only");
    if (c->fold_begin != 0 || c->fold_end != 0) throw Error(PCVG_INVALID_INPUT, "score-stream runs are unsharded");
    if (c->early_stop && (c->checkpoint_every <= 0 || c->iters % c->checkpoint_every != 0 ||
                          c->iters / c->checkpoint_every < c->blocks))
      throw Error(PCVG_INVALID_INPUT, "early_stop needs checkpoint_every dividing iters into >= blocks intervals");
    require_device(ctx);
    ctx->cfg = *cfg;
    ctx->b = effective_batch(cfg);
    ctx->fb = 0;
    ctx->fe = K;
    const int L = cfg->chains, D = sub_block_count(cfg);
    ctx->chains.clear();
    ctx->centers.clear();
    ctx->div_base.clear();
    ctx->iters_done = 0;
    ctx->sample_ms = ctx->warm_ms = 0.0;
    auto cs = std::make_unique<ChainSet>();
    cs->alloc(K * L, 1, D);
    dzero(cs->div.p, sizeof(int64_t) * cs->div.n);
    dzero(cs->pending.p, sizeof(int32_t) * cs->pending.n);
    auto cb = std::make_unique<DevBuf<double>>();
    cb->upload(std::vector<double>(centers, centers + K));
    ck(launch_centers(cs->view(L, 0, cfg->seed, 0), 0, 0, cb->p, D, ctx->stream), "reset");  // given centres
    ++ctx->launches;
    ctx->stream_scores.upload(std::vector<double>(s, s + static_cast<size_t>(K) * L * cfg->iters));
    ctx->div_base.push_back(std::vector<int64_t>(static_cast<size_t>(K) * L, 0));
    ctx->chains.push_back(std::move(cs));
    ctx->centers.push_back(std::move(cb));
    ctx->stream_mode = true;
    ctx->begun = true;
    run_checkpoints(ctx, cfg, rep);
  }));
}

}  // extern "C"

// ============================================================================ Step 1 on device
namespace {

// Model::initial_draw of each family (grouped_regression.cpp:177-188, radon.cpp:157-165,
// seasonal_ar.cpp:122-131, logistic plugin) on the chain's FullData stream (host, glibc math).
std::vector<double> initial_draw(const HostModel& m, const pcvg_model_spec* s, HostRng& rng) {
  std::vector<double> th(m.dim, 0.0);
  const int J = m.J;
  switch (m.family) {
    case PCVG_FAMILY_GROUPED: {
      const int P = m.nc;
      const double mu_a = rng.normal();
      const double sig_a = std::fabs(rng.normal()) * std::sqrt(10.0);
      const double sig_y = std::fabs(rng.normal()) * std::sqrt(10.0);
      for (int g = 0; g < J; ++g) th[g] = mu_a + sig_a * rng.normal();
      for (int p = 0; p < P; ++p) th[J + p] = rng.normal();
      th[J + P] = mu_a;
      th[J + P + 1] = std::log(sig_a);
      th[J + P + 2] = std::log(sig_y);
      break;
    }
    case PCVG_FAMILY_RADON:
      for (int g = 0; g < J; ++g) th[g] = rng.normal();
      th[J] = rng.normal();
      th[J + 1] = 2.0 * rng.normal();
      th[J + 2] = std::log(gamma_draw(rng, 6.0, 9.0));
      th[J + 3] = std::log(gamma_draw(rng, 10.0, 10.0));
      break;
    case PCVG_FAMILY_SEASONAL_AR: {
      const int p = s->ar_order, q = s->dummies;
      for (int i = 0; i < p; ++i) {
        const double w = beta_draw(rng, 5.0, 5.0);
        th[i] = std::log(w) - std::log1p(-w);
      }
      for (int j = 0; j <= q; ++j) th[p + j] = rng.normal();
      th[p + q + 1] = std::log(std::fabs(rng.normal()));
      break;
    }
    case PCVG_FAMILY_RAT_GROWTH: {  // rat_growth.cpp:228-254
      const double mu_a = 250.0 + std::sqrt(20.0) * rng.normal();
      const double mu_b = 6.0 + std::sqrt(2.0) * rng.normal();
      const double s_a = gamma_draw(rng, 25.0, 2.0);
      const double s_b = gamma_draw(rng, 5.0, 10.0);
      const double s_y = gamma_draw(rng, 1.0, 2.0);
      for (int g = 0; g < J; ++g) th[g] = mu_a + s_a * rng.normal();
      const int base = s->per_subject_slope ? 2 * J : J + 1;  // idx_mu_a (rat_growth.hpp:61)
      if (s->per_subject_slope) {
        for (int g = 0; g < J; ++g) th[J + g] = mu_b + s_b * rng.normal();
        th[base] = mu_a;
        th[base + 1] = mu_b;
        th[base + 2] = std::log(s_a);
        th[base + 3] = std::log(s_b);
        th[base + 4] = std::log(s_y);
      } else {
        th[J] = 6.0 + std::sqrt(2.0) * rng.normal();
        th[base] = mu_a;
        th[base + 1] = std::log(s_a);
        th[base + 2] = std::log(s_y);
      }
      break;
    }
    default:  // logistic plugin: independent standard normals
      for (double& t : th) t = rng.normal();
  }
  return th;
}

// DualAveraging, adapt.hpp:15-44.
struct DualAveraging {
  double target = 0.8, gamma = 0.05, t0 = 10.0, kappa = 0.75;
  double mu = 0.0, log_eps = 0.0, log_eps_bar = 0.0, h_bar = 0.0;
  long iter = 0;
  void restart(double step) {
    mu = std::log(10.0 * step);
    log_eps = std::log(step);
    log_eps_bar = log_eps;
    h_bar = 0.0;
    iter = 0;
  }
  void update(double ap) {
    ++iter;
    const double w = 1.0 / (iter + t0);
    h_bar = (1.0 - w) * h_bar + w * (target - ap);
    log_eps = mu - std::sqrt(static_cast<double>(iter)) / gamma * h_bar;
    const double w2 = std::pow(static_cast<double>(iter), -kappa);
    log_eps_bar = w2 * log_eps + (1.0 - w2) * log_eps_bar;
  }
  double current() const { return std::exp(log_eps); }
  double averaged() const { return std::exp(log_eps_bar); }
};

// StepInfo::accept_prob from the kernel's energies (hmc.cpp:79-92): 0 when divergent.
double accept_prob(double h0, double h1, int32_t flags) {
  if (flags & 2) return 0.0;
  const double dh = h1 - h0;
  return dh <= 0.0 ? 1.0 : std::exp(-dh);
}

// Chains of the adaptation: positions from the host, device streams continuing each host stream.
std::unique_ptr<ChainSet> adapt_chains(const HostModel& m, const std::vector<std::vector<double>>& pos,
                                       const std::vector<HostRng>& rngs, uint64_t stream0) {
  const int L = static_cast<int>(pos.size());
  auto cs = std::make_unique<ChainSet>();
  cs->alloc(L, m.dim, 1);
  std::vector<double> p(2 * static_cast<size_t>(m.dim) * L, 0.0);
  std::vector<uint64_t> st(L), rp(L);
  std::vector<double> cached(L);
  std::vector<int8_t> has(L);
  for (int c = 0; c < L; ++c) {
    for (int d = 0; d < m.dim; ++d) p[static_cast<size_t>(d) * L + c] = pos[c][d];
    st[c] = stream0 == 0 ? 0 : stream0;
    rp[c] = rngs[c].position();
    cached[c] = rngs[c].cached();
    has[c] = rngs[c].has_cached() ? 1 : 0;
  }
  h2d(cs->pos.p, p.data(), sizeof(double) * p.size());
  dzero(cs->grad.p, sizeof(double) * cs->grad.n);
  dzero(cs->cur.p, L);
  dzero(cs->div.p, sizeof(int64_t) * L);
  dzero(cs->warm.p, sizeof(double) * L);
  h2d(cs->rpos.p, rp.data(), sizeof(uint64_t) * L);
  h2d(cs->cached.p, cached.data(), sizeof(double) * L);
  h2d(cs->has.p, has.data(), L);
  cs->fold_override.upload(std::vector<int>(L, m.K));  // full-data sentinel fold
  return cs;
}

// param_rhat / param_ess (adapt.cpp:45-92) of parameter p over the bank [draws][L][dim].
double param_rhat(const std::vector<double>& bank, int L, int64_t n, int dim, int p) {
  double w = 0.0, grand = 0.0;
  std::vector<double> means(L);
  for (int c = 0; c < L; ++c) {
    double mm = 0.0;
    for (int64_t i = 0; i < n; ++i) mm += bank[(i * L + c) * dim + p];
    mm /= n;
    means[c] = mm;
    grand += mm / L;
    double ss = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double v = bank[(i * L + c) * dim + p];
      ss += (v - mm) * (v - mm);
    }
    w += ss / (n - 1) / L;
  }
  double b = 0.0;
  for (int c = 0; c < L; ++c) b += (means[c] - grand) * (means[c] - grand);
  b *= static_cast<double>(n) / (L - 1);
  if (!(w > 0.0)) return std::numeric_limits<double>::quiet_NaN();
  return std::sqrt(((n - 1.0) / n * w + b / n) / w);
}

double param_ess(const std::vector<double>& bank, int L, int64_t n, int dim, int p, int bsz) {
  const int64_t a = n / bsz;
  if (a < 2) return std::numeric_limits<double>::quiet_NaN();
  double grand = 0.0;
  for (int c = 0; c < L; ++c)
    for (int64_t i = 0; i < n; ++i) grand += bank[(i * L + c) * dim + p];
  grand /= static_cast<double>(L) * n;
  double ss_naive = 0.0, ss_batch = 0.0;
  for (int c = 0; c < L; ++c) {
    for (int64_t i = 0; i < n; ++i) {
      const double v = bank[(i * L + c) * dim + p];
      ss_naive += (v - grand) * (v - grand);
    }
    for (int64_t h = 0; h < a; ++h) {
      double bm = 0.0;
      for (int64_t i = h * bsz; i < (h + 1) * bsz; ++i) bm += bank[(i * L + c) * dim + p];
      bm /= bsz;
      ss_batch += (bm - grand) * (bm - grand);
    }
  }
  const double s2 = ss_naive / (static_cast<double>(L) * n - 1);
  const double sigma2 = bsz * ss_batch / (static_cast<double>(L) * a - 1);
  if (!(sigma2 > 0.0)) return std::numeric_limits<double>::quiet_NaN();
  return static_cast<double>(L) * n * s2 / sigma2;
}

}  // namespace

extern "C" pcvg_status pcvg_fold_gram(int64_t n, int32_t nc, const double* y, const double* x, const int32_t* key,
                                      int32_t K, const int32_t* lo, const int32_t* hi, double* gram) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] {
    if (n < 1 || nc < 0 || K < 0 || !y || (nc > 0 && !x) || !key || (K > 0 && (!lo || !hi)) || !gram)
      throw Error(PCVG_INVALID_INPUT, "bad fold_gram arguments");
    std::vector<int> lov(K + 1, 0), hiv(K + 1, 0);
    for (int k = 0; k < K; ++k) {
      lov[k] = lo[k];
      hiv[k] = hi[k];
    }
    SuffStats ss;
    if (!build_suffstats(n, nc, 0, y, x, key, nullptr, K, lov.data(), hiv.data(), ss, false, false))
      throw Error(PCVG_INVALID_INPUT, "non-finite data or Gram entry");
    std::copy(ss.A.begin(), ss.A.end(), gram);
  }));
}

extern "C" pcvg_status pcvg_initial_draw(const pcvg_dataset* data, const pcvg_folds* folds,
                                         const pcvg_model_spec* spec, uint64_t seed, uint64_t stream,
                                         double* theta) {
  return static_cast<pcvg_status>(guarded(nullptr, [&] {
    if (!data || !folds || !spec || !theta) throw Error(PCVG_INVALID_INPUT, "null argument");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
    // host-only: the model layout is needed for the dimensions, not the device
    HostModel m;
    m.family = spec->family;
    switch (spec->family) {
      case PCVG_FAMILY_GROUPED: m.J = n_groups(data); m.nc = data->n_cov; m.ng = data->n_cov + 3; break;
      case PCVG_FAMILY_RADON: m.J = n_groups(data); m.nc = 1; m.ng = 4; break;
      case PCVG_FAMILY_SEASONAL_AR: m.J = 0; m.nc = spec->ar_order + spec->dummies; m.ng = m.nc + 2; break;
      case PCVG_FAMILY_LOGISTIC: m.J = 0; m.nc = data->n_cov; m.ng = data->n_cov + 1; break;
      case PCVG_FAMILY_RAT_GROWTH: m.J = n_groups(data); m.nc = 1; m.ng = spec->per_subject_slope ? 5 : 4; break;
      default: throw Error(PCVG_INVALID_INPUT, "model family not available");
    }
    m.dim = m.J * ((spec->family == PCVG_FAMILY_RAT_GROWTH && spec->per_subject_slope) ? 2 : 1) + m.ng;
    HostRng rng(seed, stream);
    const auto th = initial_draw(m, spec, rng);
    std::copy(th.begin(), th.end(), theta);
    (void)folds;
    (void)count;
  }));
}

extern "C" pcvg_status pcvg_adapt_full_data(pcvg_ctx* ctx, const pcvg_dataset* data,
                                            const pcvg_folds* folds, const pcvg_model_spec* spec,
                                            const pcvg_adapt_config* cfg, uint64_t seed,
                                            int32_t model_id, pcvg_fit* out) {
  return static_cast<pcvg_status>(guarded(ctx, [&] {
    if (!ctx || !cfg || !out || !data || !spec) throw Error(PCVG_INVALID_INPUT, "null argument");
    if (cfg->chains < 1 || cfg->warmup < 1 || cfg->draws < 1)  // adapt.cpp:97-99
      throw Error(PCVG_INVALID_INPUT, "full-data config needs chains, warmup, draws >= 1");
    if (cfg->n_leapfrog < 1) throw Error(PCVG_INVALID_INPUT, "n_leapfrog must be >= 1");
    if (cfg->chains > 64) throw Error(PCVG_INVALID_INPUT, "at most 64 full-data chains on device");
    if (!out->inv_mass_diag || !out->draws) throw Error(PCVG_INVALID_INPUT, "fit output buffers missing");
    require_device(ctx);
    // the model in device layout; kernel and bank are placeholders until adapted
    const int dim_cap = (data->group_id ? 2 * n_groups(data) : 0) + data->n_cov + 8;
    std::vector<double> ones(dim_cap, 1.0), zero(dim_cap, 0.0);
    pcvg_kernel k0{1.0, cfg->n_leapfrog, ones.data()};
    auto hm = build_model(data, folds, spec, &k0, zero.data(), 1, model_id);
    const HostModel& m = *hm;
    const int d = m.dim, L = cfg->chains;
    if (d < 1) throw Error(PCVG_INVALID_INPUT, "model has no parameters");
    ModelDev md = m.md;
    DevBuf<double> im;
    std::vector<double> inv_mass(d, 1.0);
    im.upload(inv_mass);
    md.inv_mass = im.p;
    md.n_lf = cfg->n_leapfrog;

    // chains from the prior on their FullData streams (adapt.cpp:104-110)
    std::vector<std::vector<double>> pos;
    std::vector<HostRng> rngs;
    for (int c = 0; c < L; ++c) {
      HostRng rng(seed, stream_key(PCVG_STREAM_FULL_DATA, static_cast<uint64_t>(model_id),
                                   static_cast<uint64_t>(c), 0));
      pos.push_back(initial_draw(m, spec, rng));
      rngs.push_back(rng);
    }
    auto cs = adapt_chains(m, pos, rngs, 0);
    {
      std::vector<uint64_t> st(L);
      for (int c = 0; c < L; ++c)
        st[c] = stream_key(PCVG_STREAM_FULL_DATA, static_cast<uint64_t>(model_id), static_cast<uint64_t>(c), 0);
      h2d(cs->stream.p, st.data(), sizeof(uint64_t) * L);
    }
    const ChainsDev S = cs->view(1, 0, seed, 0);
    DevBuf<double> h0b, h1b;
    DevBuf<int32_t> flb;
    DevBuf<double> trb;
    float ms_total = 0.f;
    auto trace = [&](const ChainSet& set, const ChainsDev& SS, int64_t n_iters, bool positions,
                     std::vector<double>& h0, std::vector<double>& h1, std::vector<int32_t>& fl,
                     std::vector<double>* traj) {
      const size_t rows = static_cast<size_t>(n_iters) * SS.nch;
      if (h0b.n < rows) { h0b.alloc(rows); h1b.alloc(rows); flb.alloc(rows); }
      if (positions && trb.n < rows * d) trb.alloc(rows * d);
      RunArgs a = make_args(kModeChain, n_iters);
      a.out_a = h0b.p;
      a.out_b = h1b.p;
      a.traj_div = flb.p;
      a.traj = positions ? trb.p : nullptr;
      ck(cudaEventRecord(ctx->ev0, ctx->stream), "event");
      launch_family(ctx, m, SS, a, ctx->stream, &md);
      ck(cudaEventRecord(ctx->ev1, ctx->stream), "event");
      ck(cudaEventSynchronize(ctx->ev1), "adapt");
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
      ms_total += ms;
      h0.resize(rows);
      h1.resize(rows);
      fl.resize(rows);
      ck(cudaMemcpy(h0.data(), h0b.p, sizeof(double) * rows, cudaMemcpyDeviceToHost), "download");
      ck(cudaMemcpy(h1.data(), h1b.p, sizeof(double) * rows, cudaMemcpyDeviceToHost), "download");
      ck(cudaMemcpy(fl.data(), flb.p, sizeof(int32_t) * rows, cudaMemcpyDeviceToHost), "download");
      if (positions && traj) {
        traj->resize(rows * d);
        ck(cudaMemcpy(traj->data(), trb.p, sizeof(double) * rows * d, cudaMemcpyDeviceToHost), "download");
      }
      (void)set;
    };
    std::vector<double> h0, h1, tr;
    std::vector<int32_t> fl;

    // first step size: doubling search on chain 0's start (adapt.cpp:17-43)
    double step = cfg->init_step_size;
    if (!(step > 0.0)) {
      const uint64_t sst = stream_key(PCVG_STREAM_STEP_INIT, static_cast<uint64_t>(model_id), 0, 0);
      auto probe = [&](double e) {
        HostRng fresh(seed, sst);
        auto ps = adapt_chains(m, {pos[0]}, {fresh}, 0);
        h2d(ps->stream.p, &sst, sizeof sst);
        ModelDev saved = md;
        md.step = e;
        md.n_lf = 1;
        const ChainsDev PS = ps->view(1, 0, seed, 0);
        launch_family(ctx, m, PS, make_args(kModeEval, 0), ctx->stream, &md);
        trace(*ps, PS, 1, false, h0, h1, fl, nullptr);
        md = saved;
        return accept_prob(h0[0], h1[0], fl[0]);
      };
      double eps = 1.0;
      const bool go_up = probe(eps) > 0.5;
      bool done = false;
      for (int i = 0; i < 50 && !done; ++i) {
        if (go_up) {
          eps *= 2.0;
          if (probe(eps) <= 0.5) { eps /= 2.0; done = true; }
        } else {
          eps *= 0.5;
          if (probe(eps) > 0.5) done = true;
        }
      }
      step = done ? eps : (go_up ? eps : 1e-8);
    }
    md.step = step;
    launch_family(ctx, m, S, make_args(kModeEval, 0), ctx->stream, &md);  // grad / lp0 at the starts

    // windowed adaptation (adapt.cpp:112-185)
    DualAveraging da;
    da.target = cfg->target_accept;
    da.restart(step);
    const int64_t w_total = cfg->warmup;
    const int64_t w_init = std::min<int64_t>(75, std::max<int64_t>(1, w_total * 15 / 100));
    const int64_t w_final = std::min<int64_t>(50, std::max<int64_t>(1, w_total / 10));
    int64_t window = 25;
    int64_t window_end = std::min(w_total - w_final, w_init + window);
    std::vector<double> wx(d, 0.0), wx2(d, 0.0);  // WelfordDiag(d), centre 0 (accum.cpp:59-74)
    int64_t wcount = 0;
    int64_t window_div = 0, window_steps = 0;
    for (int64_t iter = 0; iter < w_total; ++iter) {
      md.step = da.current();
      if (out->step_trace) out->step_trace[iter] = md.step;
      const bool in_slow = iter >= w_init && iter < w_total - w_final;
      trace(*cs, S, 1, in_slow, h0, h1, fl, &tr);
      double ap = 0.0;
      int64_t n_div = 0;
      for (int c = 0; c < L; ++c) {
        ap += accept_prob(h0[c], h1[c], fl[c]);
        n_div += (fl[c] >> 1) & 1;
      }
      ap /= L;
      da.update(ap);
      window_div += n_div;
      window_steps += L;
      if (in_slow) {
        for (int c = 0; c < L; ++c)
          for (int i = 0; i < d; ++i) {
            const double v = tr[static_cast<size_t>(c) * d + i];
            wx[i] += v;
            wx2[i] += v * v;
          }
        wcount += L;
      }
      if (in_slow && iter + 1 == window_end) {
        if (wcount >= 2) {
          const double n = static_cast<double>(wcount);
          for (int i = 0; i < d; ++i) {
            const double var = (wx2[i] - wx[i] * wx[i] / wcount) / (wcount - 1);
            const double v = var * (n / (n + 5.0)) + 1e-3 * (5.0 / (n + 5.0));
            inv_mass[i] = std::max(v, 1e-10);
          }
          h2d(im.p, inv_mass.data(), sizeof(double) * d);
        }
        std::fill(wx.begin(), wx.end(), 0.0);
        std::fill(wx2.begin(), wx2.end(), 0.0);
        wcount = 0;
        da.restart(da.current());
        window *= 2;
        int64_t next_end = window_end + window;
        if (next_end + 2 * window > w_total - w_final) next_end = w_total - w_final;
        window_end = next_end;
      }
      if (window_steps >= 100 * L) {  // persistent-failure check (adapt.cpp:169-180)
        if (window_div > window_steps / 2)
          throw Error(PCVG_ADAPTATION_FAILURE, "full-data adaptation failed: chains diverging persistently");
        window_div = 0;
        window_steps = 0;
      }
    }
    md.step = da.averaged();

    // frozen-kernel draws fill the bank (adapt.cpp:194-210), one launch
    trace(*cs, S, cfg->draws, true, h0, h1, fl, &tr);
    double acc = 0.0;
    int64_t ndiv = 0;
    for (size_t r = 0; r < h0.size(); ++r) {
      acc += accept_prob(h0[r], h1[r], fl[r]);
      ndiv += (fl[r] >> 1) & 1;
    }
    out->step_size = md.step;
    std::copy(inv_mass.begin(), inv_mass.end(), out->inv_mass_diag);
    std::copy(tr.begin(), tr.end(), out->draws);
    out->divergences = ndiv;
    out->mean_accept = acc / (static_cast<double>(L) * cfg->draws);
    const int ess_b = std::max(1, static_cast<int>(std::sqrt(static_cast<double>(cfg->draws))));
    for (int p = 0; p < d; ++p) {
      if (out->rhat) out->rhat[p] = L >= 2 ? param_rhat(tr, L, cfg->draws, d, p) : std::numeric_limits<double>::quiet_NaN();
      if (out->ess) out->ess[p] = param_ess(tr, L, cfg->draws, d, p, ess_b);
    }
    out->device_ms = ms_total;
  }));
}
