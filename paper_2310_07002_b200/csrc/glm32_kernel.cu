// FP32 variant of the logistic HMC kernel on the 5th-generation tensor cores (sm_100a), the
// "FP32 variant reported separately" of SURVEY 8(d): the two contractions of every gradient pass,
//   eta = X . Theta        (128 rows x 64 chains, K = 56)
//   G   = X^T . R          (56 columns x 64 chains, K = 128 rows per tile)
// run as tcgen05.mma kind::tf32 with both operands split exactly into a TF32 high part and an FP32
// remainder (x = hi + lo, hi = round-to-TF32(x)); all four products are accumulated in FP32 in
// tensor memory, which gives FP32-class accuracy (per-step gradients within 1e-5 of the FP64
// path, the north star's FP32 tolerance). The split is folded into the operand shapes instead of
// extra instructions:
//   eta: B = [Theta_hi | Theta_lo] (N = 128), issued once with A = X_hi and once with A = X_lo;
//        eta = D[:, c] + D[:, 64 + c].
//   G:   A = [X_hi^T ; X_lo^T] (M = 128 stacked columns), issued once with B = R_hi and once with
//        B = R_lo; G = D[k, :] + D[56 + k, :].
// Every operand is K-major (SWIZZLE_NONE canonical layout, 16-byte core rows of 4 TF32 values), so
// each 128-row tile of the design has two host-built images: the eta image ([16-byte column chunk]
// [row][4], hi then lo) and the G image ([16-byte row chunk][stacked column][4]). They stream by
// TMA bulk copies into two single buffers that are refilled as soon as the MMA reading them has
// completed (the eta image during the epilogue and G, the G image during the next eta), with y and
// the row keys double-buffered beside the eta image. Since the design does not depend on theta,
// the copies run ahead across gradient passes. One elected thread issues the MMAs and commits them
// to mbarriers; all 16 warps drain TMEM (warp w reads lane quadrant w%4, chain group w/4),
// evaluate the sigmoid and the mask in FP32, and write R_hi / R_lo in the B layout of G. G is
// flushed from TMEM into FP64 per-CTA accumulators every 16 tiles. The chain
// state, integrator, energies, Metropolis test, RNG, log_pred and accumulators are FP64 and the
// same as glm_kernel.cu (hmc.cpp:22-99, engine.cpp:342-381).
#include <math_constants.h>

#include <cstdint>
#include <cstring>

#include "device_common.cuh"
#include "tc_common.cuh"
#include "types.cuh"

namespace pcvg {

namespace {

using namespace tc;

constexpr int kC = 64;                          // chains per CTA
constexpr int kThreads = 512;                   // 16 warps
constexpr int kOwners = kThreads / kC;          // owner threads per chain
constexpr int kRows = 128;                      // rows per tile = UMMA M of eta = TMEM lanes
constexpr int kK = 56;                          // padded design width (1 + 50 covariates + pad)
constexpr int kChunks = kK / 4;                 // 16-byte column chunks per row
constexpr int kOwn = (kK + kOwners - 1) / kOwners;
constexpr int kChunkBytes = kRows * 16;         // one column chunk of a tile image (2048)
constexpr int kXImg = 2 * kChunks * kChunkBytes;  // eta image: hi + lo (57344)
constexpr int kYK = kRows * 8;                  // y (f32) + key (i32)
constexpr int kGImg = (kRows / 4) * 128 * 16;   // G image: [row chunk][128 stacked columns][4] (65536)
constexpr int kTileBytes = kXImg + kYK + kGImg; // per tile in HBM: eta image, y/key, G image
constexpr int kRLbo = kC * 16 + 16;             // R image chunk stride: +16 B keeps the stores conflict-free
constexpr int kRImg = (kRows / 4) * kRLbo;
constexpr int kThImg = kChunks * 2 * kC * 16;   // [chunk][hi chains | lo chains][4]
constexpr int kFlush = 16;                      // tiles between FP32 -> FP64 flushes of G
constexpr uint32_t kTmemCols = 256;             // eta: 128 columns, G: 64 columns
constexpr uint32_t kEtaCol = 0, kGCol = 128;

static_assert(kTileBytes % 16 == 0 && kXImg % 16 == 0 && kYK % 16 == 0, "bulk copy granularity");
static_assert(2 * kK <= 128, "stacked hi/lo columns fit one M = 128 operand");

struct Smem32 {
  alignas(128) unsigned char xa[kXImg];
  alignas(128) unsigned char yk[2][kYK];
  alignas(128) unsigned char xb[kGImg];
  alignas(128) unsigned char th[kThImg];
  alignas(128) unsigned char r[2][kRImg];
  double red[kOwners][kC];
  double pri[kOwners][kC];
  double llq[4][kC];
  int lo[kC], hi[kC], ntr[kC], bad[kC], cur[kC];
  unsigned long long full_a, full_b, full_y[2];  // eta image, G image, y/key slots
  unsigned long long mma_eta, mma_g;
  uint32_t tmem_base;
};

static_assert(sizeof(Smem32) <= 232448, "fits the 227 KB opt-in shared memory of one CTA");

// ------------------------------------------------------------------ tcgen05 helpers
// Shared-memory matrix descriptor (SWIZZLE_NONE canonical layout, sm_100 version bits).
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  const uint64_t a = (smem_addr(p) >> 4) & 0x3FFFu;
  return a | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// Instruction descriptor: kind::tf32, FP32 accumulate, M x N, operand majors (0 = K, 1 = MN).
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc ? 1 : 0));
}

__device__ __forceinline__ void mma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

// 16 consecutive 32-bit TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void split_store(unsigned char* hi_img, unsigned char* lo_img, uint32_t off, float v) {
  const float h = tf32_hi(v);
  *reinterpret_cast<float*>(hi_img + off) = h;
  *reinterpret_cast<float*>(lo_img + off) = v - h;
}

__device__ __forceinline__ double bernoulli_logit32(double y, double x) {
  return y * x - (fmax(x, 0.0) + log1p(exp(-fabs(x))));
}

// ------------------------------------------------------------------ one gradient pass
// Tile stream state: g = tiles consumed so far (over all passes), ia / ib = eta / G images issued.
// Load j carries tile j % ntiles; the eta image buffer, the G image buffer and each y/key slot see
// their loads complete in order, so the mbarrier parity of load j is j & 1 (y/key: (j >> 1) & 1).
struct Pipe32 {
  uint32_t g = 0, ia = 0, ib = 0, n_eta = 0, n_g = 0;
};

__device__ __forceinline__ const unsigned char* tile_src(const ModelDev& M, uint32_t j, int ntiles) {
  return M.x32 + static_cast<size_t>(j % static_cast<uint32_t>(ntiles)) * kTileBytes;
}
__device__ __forceinline__ void load_eta_image(Smem32& sm, const ModelDev& M, uint32_t j, int ntiles) {
  const unsigned char* src = tile_src(M, j, ntiles);
  fence_proxy_async();
  mbar_expect_tx(&sm.full_a, kXImg);
  bulk_g2s(sm.xa, src, kXImg, &sm.full_a);
  mbar_expect_tx(&sm.full_y[j & 1], kYK);
  bulk_g2s(sm.yk[j & 1], src + kXImg, kYK, &sm.full_y[j & 1]);
}
__device__ __forceinline__ void load_g_image(Smem32& sm, const ModelDev& M, uint32_t j, int ntiles) {
  fence_proxy_async();
  mbar_expect_tx(&sm.full_b, kGImg);
  bulk_g2s(sm.xb, tile_src(M, j, ntiles) + kXImg + kYK, kGImg, &sm.full_b);
}

// Accumulates G (FP64, [stacked column m][chain] in gsc) over all tiles for the CTA's 64 chains
// with the parameters in the theta image; VALUE adds the per-chain log-likelihood into sm.llq.
// `more` = another pass follows (its first tile may be prefetched).
template <bool VALUE>
__device__ void grad_pass32(Smem32& sm, const ModelDev& M, double* gsc, Pipe32& P, int ntiles, bool more) {
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int qd = w & 3, cg = w >> 2;  // TMEM lane quadrant, chain group (16 chains)
  const uint32_t tmem = sm.tmem_base;
  const uint32_t lane_off = static_cast<uint32_t>(32 * qd) << 16;
  constexpr uint32_t kIdEta = idesc_tf32(128, 128, 0, 0);
  constexpr uint32_t kIdG = idesc_tf32(128, 64, 0, 0);
  if (VALUE) {
    for (int i = tid; i < 4 * kC; i += kThreads) (&sm.llq[0][0])[i] = 0.0;
    __syncthreads();
  }
  if (tid == 0) {  // first tile of the pass, unless the previous pass prefetched it
    if (P.ia == P.g) load_eta_image(sm, M, P.ia++, ntiles);
    if (P.ib == P.g) load_g_image(sm, M, P.ib++, ntiles);
  }
  bool first_flush = true;
  for (int t = 0; t < ntiles; ++t) {
    const uint32_t g = P.g + t;
    const bool next = t + 1 < ntiles || more;
    // ---- eta = X . [Th_hi | Th_lo]  (7 k-steps x {X_hi, X_lo})
    if (tid == 0) {
      mbar_wait(&sm.full_a, g & 1u);
      tmem_fence_after();
      for (int half = 0; half < 2; ++half)
        for (int ks = 0; ks < kChunks / 2; ++ks) {
          const uint64_t a = sdesc(sm.xa + (half * kChunks + 2 * ks) * kChunkBytes, kChunkBytes, 128);
          const uint64_t b = sdesc(sm.th + 2 * ks * (2 * kC * 16), 2 * kC * 16, 128);
          mma_tf32(tmem + kEtaCol, a, b, kIdEta, half > 0 || ks > 0);
        }
      mma_commit(&sm.mma_eta);
    }
    mbar_wait(&sm.mma_eta, P.n_eta & 1u);
    ++P.n_eta;
    if (tid == 0 && next) load_eta_image(sm, M, P.ia++, ntiles);  // eta(g) done: the buffer is free
    mbar_wait(&sm.full_y[g & 1], (g >> 1) & 1u);
    tmem_fence_after();
    // ---- residuals of this warp's 32 rows x 16 chains
    {
      float eh[16], el[16];
      tmem_ld16(tmem + lane_off + kEtaCol + 16 * cg, eh);
      tmem_ld16(tmem + lane_off + kEtaCol + kC + 16 * cg, el);
      const int r = 32 * qd + l;
      const float yv = reinterpret_cast<const float*>(sm.yk[g & 1])[r];
      const int kv = reinterpret_cast<const int*>(sm.yk[g & 1] + kRows * 4)[r];
      const uint32_t roff = (r >> 2) * kRLbo + (r & 3) * 4;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = 16 * cg + j;
        const float eta = eh[j] + el[j];
        const bool real = kv >= 0;
        const bool train = real && static_cast<unsigned>(kv - sm.lo[c]) >= static_cast<unsigned>(sm.hi[c] - sm.lo[c]);
        const float sig = 1.0f / (1.0f + __expf(-eta));
        const float res = train ? yv - sig : 0.0f;
        split_store(sm.r[0], sm.r[1], roff + c * 16, res);
        if (VALUE) {
          float ll = 0.0f;
          if (train) ll = yv * eta - (fmaxf(eta, 0.0f) + log1pf(__expf(-fabsf(eta))));
          else if (real && !isfinite(eta)) ll = CUDART_NAN_F;  // 0 * non-finite test term
          for (int o = 16; o > 0; o >>= 1) ll += __shfl_xor_sync(0xffffffffu, ll, o);
          if (l == 0) sm.llq[qd][c] += static_cast<double>(ll);
        }
      }
    }
    tmem_fence_before();
    fence_proxy_async();  // R image writes before the async-proxy MMA reads them
    __syncthreads();
    // ---- G += [X_hi^T ; X_lo^T] . R_hi + ... . R_lo  (16 k-steps of 8 rows)
    const bool fresh = t % kFlush == 0;
    if (tid == 0) {
      mbar_wait(&sm.full_b, g & 1u);
      tmem_fence_after();
      for (int ks = 0; ks < kRows / 8; ++ks) {
        const uint64_t a = sdesc(sm.xb + 2 * ks * 2048, 2048, 128);
        const uint64_t b0 = sdesc(sm.r[0] + 2 * ks * kRLbo, kRLbo, 128);
        const uint64_t b1 = sdesc(sm.r[1] + 2 * ks * kRLbo, kRLbo, 128);
        mma_tf32(tmem + kGCol, a, b0, kIdG, !(fresh && ks == 0));
        mma_tf32(tmem + kGCol, a, b1, kIdG, true);
      }
      mma_commit(&sm.mma_g);
    }
    mbar_wait(&sm.mma_g, P.n_g & 1u);
    ++P.n_g;
    if (tid == 0 && next) load_g_image(sm, M, P.ib++, ntiles);  // G(g) done: the buffer is free
    const bool flush = (t + 1) % kFlush == 0 || t + 1 == ntiles;
    if (flush) {  // G (FP32, TMEM) -> FP64 accumulators [m][chain]
      tmem_fence_after();
      float gv[16];
      tmem_ld16(tmem + lane_off + kGCol + 16 * cg, gv);
      const int m = 32 * qd + l;
      if (m < 2 * kK) {
        double* dst = gsc + static_cast<size_t>(m) * kC + 16 * cg;
#pragma unroll
        for (int j = 0; j < 16; ++j) dst[j] = first_flush ? static_cast<double>(gv[j]) : dst[j] + static_cast<double>(gv[j]);
      }
      first_flush = false;
      tmem_fence_before();
    }
    __syncthreads();  // eta / R buffers and the G accumulator are reused by the next tile
  }
  P.g += ntiles;
}

__global__ void __launch_bounds__(kThreads, 1) glm32_kernel(ModelDev M, ChainsDev S, RunArgs A, double* gscratch) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem32& sm = *reinterpret_cast<Smem32*>(smem_raw);
  const int tid = threadIdx.x;
  const int nch = S.nch;
  const int dim = M.dim;
  const size_t plane = static_cast<size_t>(dim) * nch;
  const int tile = blockIdx.x;
  const int ntiles = (M.n + kRows - 1) / kRows;
  const int oc = tid & (kC - 1), ok = tid / kC;
  const int ogc = tile * kC + oc;
  const bool ovalid = ogc < nch;
  const bool is_chain = tid < kC;
  const int gc = tile * kC + tid;
  const bool cvalid = is_chain && gc < nch;
  double* gsc = gscratch + static_cast<size_t>(blockIdx.x) * (2 * kK) * kC;

  if (tid == 0) mbar_init(&sm.full_a, 1);
  if (tid == 1) mbar_init(&sm.full_b, 1);
  if (tid == 2) mbar_init(&sm.mma_eta, 1);
  if (tid == 3) mbar_init(&sm.mma_g, 1);
  if (tid == 4 || tid == 5) mbar_init(&sm.full_y[tid - 4], 1);
  fence_mbar_init();
  if (tid < 32) {  // warp 0 allocates the tensor memory
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(&sm.tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  ChainRng R;
  double lp0 = 0.0, warm = 0.0;
  int64_t div_count = 0;
  int fold = M.K;
  if (is_chain) {
    if (cvalid) {
      fold = S.fold_override ? S.fold_override[gc] : S.fold0 + gc / S.L;
      sm.lo[tid] = M.fold_lo[fold];
      sm.hi[tid] = M.fold_hi[fold];
      sm.ntr[tid] = M.n_train[fold];
      sm.cur[tid] = S.cur[gc];
      lp0 = S.lp0[gc];
      R.init(S.seed, S.rng_stream[gc], S.rng_pos[gc], S.rng_cached[gc], S.rng_has[gc] != 0);
    } else {
      sm.lo[tid] = 0;
      sm.hi[tid] = 0;
      sm.ntr[tid] = M.n;
      sm.cur[tid] = 0;
    }
  }
  for (int i = tid; i < kThImg / 4; i += kThreads) reinterpret_cast<float*>(sm.th)[i] = 0.0f;
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  Pipe32 P;

  double qown[kOwn];
  // owners publish theta (hi / lo) into the B image of eta: element (n, k) at
  // (k/4) * (2 kC 16) + n * 16 + (k%4) * 4, n = chain (hi) or kC + chain (lo)
  auto put_theta = [&]() {
#pragma unroll
    for (int j = 0; j < kOwn; ++j) {
      const int k = ok + kOwners * j;
      if (k < dim) {
        const float v = static_cast<float>(qown[j]);
        const float h = tf32_hi(v);
        const uint32_t off = (k >> 2) * (2 * kC * 16) + (k & 3) * 4;
        *reinterpret_cast<float*>(sm.th + off + oc * 16) = h;
        *reinterpret_cast<float*>(sm.th + off + (kC + oc) * 16) = v - h;
      }
    }
    fence_proxy_async();
  };
  auto gk_of = [&](int k) { return gsc[static_cast<size_t>(k) * kC + oc] + gsc[static_cast<size_t>(kK + k) * kC + oc]; };
  auto ll_of = [&](int c) { return (sm.llq[0][c] + sm.llq[1][c]) + (sm.llq[2][c] + sm.llq[3][c]); };
  auto lp_from_partials = [&](int c) {
    double pr = 0.0;
#pragma unroll
    for (int o = 0; o < kOwners; ++o) pr += sm.pri[o][c];
    return ll_of(c) + pr;
  };

  if (A.mode == kModeEval) {
    const int cu = sm.cur[oc];
#pragma unroll
    for (int j = 0; j < kOwn; ++j) {
      const int k = ok + kOwners * j;
      qown[j] = (k < dim && ovalid) ? S.pos[cu * plane + static_cast<size_t>(k) * nch + ogc] : 0.0;
    }
    put_theta();
    __syncthreads();
    grad_pass32<true>(sm, M, gsc, P, ntiles, false);
    double pr = 0.0;
#pragma unroll
    for (int j = 0; j < kOwn; ++j) {
      const int k = ok + kOwners * j;
      if (k < dim) {
        if (ovalid) S.grad[cu * plane + static_cast<size_t>(k) * nch + ogc] = gk_of(k) - qown[j];
        pr += -0.5 * (kLog2Pi + qown[j] * qown[j]);
      }
    }
    sm.pri[ok][oc] = pr;
    __syncthreads();
    if (cvalid) {
      const double lp = lp_from_partials(tid);
      S.lp0[gc] = lp;
      if (A.out_a) A.out_a[gc] = lp;
    }
  } else {
    const double eps = M.step, half = 0.5 * M.step;
    const int n_lf = M.n_lf;
    for (int64_t it = 0; it < A.n_iters; ++it) {
      if (A.mode != kModePred) {
        // momentum refresh (chain thread, reference draw order) -> staging in sm.red/pri? use R image
        double k0 = 0.0;
        double* pstage = reinterpret_cast<double*>(sm.r[0]);  // [k][chain], free between passes
        if (is_chain) {
          for (int k = 0; k < dim; ++k) {
            const double mk = __ldg(M.inv_mass + k);
            double p;
            if (A.mode == kModeProbe) p = cvalid ? A.probe_momentum[static_cast<size_t>(gc) * dim + k] : 0.0;
            else p = R.normal() / sqrt(mk);
            k0 += mk * p * p;
            pstage[k * kC + tid] = p;
          }
          sm.bad[tid] = 0;
        }
        __syncthreads();
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
              p = pstage[k * kC + oc] + half * S.grad[gi];
              q = S.pos[gi] + eps * __ldg(M.inv_mass + k) * p;
              bad |= !isfinite(q);
            }
            qown[j] = q;
            pown[j] = p;
          }
          if (bad) sm.bad[oc] = 1;
        }
        __syncthreads();  // momentum staging read before the R images are overwritten
        put_theta();
        __syncthreads();
        for (int s = 0; s < n_lf; ++s) {
          const bool last = s == n_lf - 1;
          const bool more = !last || it + 1 < A.n_iters;
          if (last) grad_pass32<true>(sm, M, gsc, P, ntiles, more);
          else grad_pass32<false>(sm, M, gsc, P, ntiles, more);
          const double scale = last ? half : eps;
          const int cu = sm.cur[oc];
          bool bad = false;
          double part = 0.0, part2 = 0.0;
#pragma unroll
          for (int j = 0; j < kOwn; ++j) {
            const int k = ok + kOwners * j;
            if (k < dim) {
              const double g = gk_of(k) - qown[j];
              bad |= !isfinite(g);
              pown[j] += scale * g;
              bad |= !isfinite(pown[j]);
              if (last) {
                part += __ldg(M.inv_mass + k) * pown[j] * pown[j];
                part2 += -0.5 * (kLog2Pi + qown[j] * qown[j]);
                if (ovalid) {
                  const size_t gi = (cu ^ 1) * plane + static_cast<size_t>(k) * nch + ogc;
                  S.pos[gi] = qown[j];
                  S.grad[gi] = g;
                  if (A.mode == kModeProbe && A.traj) A.traj[static_cast<size_t>(ogc) * dim + k] = pown[j];
                }
              } else {
                qown[j] += eps * __ldg(M.inv_mass + k) * pown[j];
                bad |= !isfinite(qown[j]);
              }
            }
          }
          if (last) {
            sm.red[ok][oc] = part;
            sm.pri[ok][oc] = part2;
          }
          if (bad) sm.bad[oc] = 1;
          __syncthreads();  // G scratch read by every owner before the next pass rewrites it
          if (!last) {
            put_theta();
            __syncthreads();
          }
        }
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
          if (cvalid && A.mode == kModeChain) {
            const size_t row = static_cast<size_t>(it) * nch + gc;
            if (A.traj_div) A.traj_div[row] = (accepted ? 1 : 0) | (divergent ? 2 : 0);
            if (A.out_a) A.out_a[row] = h0;
            if (A.out_b) A.out_b[row] = h1;
          }
        }
        __syncthreads();
        if (A.mode == kModeProbe) continue;
        if (A.mode == kModeChain) {
          const int cu = sm.cur[oc];
          if (ovalid && A.traj) {
#pragma unroll
            for (int j = 0; j < kOwn; ++j) {
              const int k = ok + kOwners * j;
              if (k < dim)
                A.traj[(static_cast<size_t>(it) * nch + ogc) * dim + k] = S.pos[cu * plane + static_cast<size_t>(k) * nch + ogc];
            }
          }
          continue;
        }
      }
      // log_pred (FP64) at the current position + accumulators (engine.cpp:360-373)
      if (cvalid) {
        double sp = 0.0;
        if (fold < M.K) {
          const double* pos = S.pos + sm.cur[tid] * plane + gc;
          const int s0 = M.fold_seg[fold], s1 = M.fold_seg[fold + 1];
          for (int sg = s0; sg < s1; ++sg)
            for (int tt = M.seg_row[sg]; tt < M.seg_row[sg + 1]; ++tt) {
              const int i = M.seg_rows[tt];
              const double* xrow = M.xr + static_cast<size_t>(i) * M.nc_pad;
              double eta = 0.0;
              for (int k = 0; k < dim; ++k) eta = fma(xrow[k], pos[static_cast<size_t>(k) * nch], eta);
              sp += bernoulli_logit32(M.y[i], eta);
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
  if (tid == 0) {  // no bulk copy may still be landing in shared memory at exit
    if (P.ia > P.g) {
      mbar_wait(&sm.full_a, P.g & 1u);
      mbar_wait(&sm.full_y[P.g & 1], (P.g >> 1) & 1u);
    }
    if (P.ib > P.g) mbar_wait(&sm.full_b, P.g & 1u);
  }
  tmem_fence_before();
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(sm.tmem_base), "r"(kTmemCols));
}

}  // namespace

// Bytes of the FP32 tile images of an n-row logistic design (glm32_tile_image).
size_t glm32_image_bytes(int64_t n) { return static_cast<size_t>((n + kRows - 1) / kRows) * kTileBytes; }

// Host: the tile images of the augmented design xr ([n][KP] row-major, column 0 = intercept). Per
// 128-row tile: the eta image [hi: 14 chunks][lo: 14 chunks] x [128 rows][4 columns], y (FP32), the
// row key (int32, -1 on padding rows), then the G image [32 row chunks][128 stacked columns: hi 0..55,
// lo 56..111, zero 112..127][4 rows].
void glm32_tile_image(const double* xr, int kp, const double* y, const int* key, int64_t n, unsigned char* out) {
  const int64_t ntiles = (n + kRows - 1) / kRows;
  for (int64_t t = 0; t < ntiles; ++t) {
    unsigned char* img = out + t * kTileBytes;
    std::memset(img, 0, kTileBytes);
    float* hi = reinterpret_cast<float*>(img);
    float* lo = reinterpret_cast<float*>(img + kXImg / 2);
    float* ys = reinterpret_cast<float*>(img + kXImg);
    int* ks = reinterpret_cast<int*>(img + kXImg + kRows * 4);
    float* gi = reinterpret_cast<float*>(img + kXImg + kYK);
    for (int r = 0; r < kRows; ++r) {
      const int64_t i = t * kRows + r;
      for (int k = 0; k < kK; ++k) {
        const float v = (i < n && k < kp) ? static_cast<float>(xr[i * kp + k]) : 0.0f;
        uint32_t bits;
        std::memcpy(&bits, &v, 4);
        // round to nearest TF32 (10 explicit mantissa bits), ties away from zero like cvt.rna
        uint32_t hb = (bits + 0x1000u) & 0xFFFFE000u;
        if ((bits & 0x7F800000u) == 0x7F800000u) hb = bits;
        float h;
        std::memcpy(&h, &hb, 4);
        const size_t off = static_cast<size_t>(k / 4) * kRows * 4 + r * 4 + (k % 4);
        hi[off] = h;
        lo[off] = v - h;
        const size_t go = static_cast<size_t>(r / 4) * 128 * 4 + (r % 4);
        gi[go + static_cast<size_t>(k) * 4] = h;
        gi[go + static_cast<size_t>(kK + k) * 4] = v - h;
      }
      ys[r] = i < n ? static_cast<float>(y[i]) : 0.0f;
      ks[r] = i < n ? key[i] : -1;
    }
  }
}

cudaError_t launch_glm32(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st) {
  const int tiles = (S.nch + kC - 1) / kC;
  if (tiles == 0) return cudaSuccess;
  if (M.family != kLogistic || M.x32 == nullptr || M.dim > kK) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(glm32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sizeof(Smem32)));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  static double* scratch = nullptr;
  static int scratch_tiles = 0;
  if (tiles > scratch_tiles) {
    if (scratch) cudaFree(scratch);
    cudaError_t e = cudaMalloc(&scratch, sizeof(double) * static_cast<size_t>(tiles) * 2 * kK * kC);
    if (e != cudaSuccess) return e;
    scratch_tiles = tiles;
  }
  glm32_kernel<<<tiles, kThreads, sizeof(Smem32), st>>>(M, S, A, scratch);
  return cudaGetLastError();
}

}  // namespace pcvg
