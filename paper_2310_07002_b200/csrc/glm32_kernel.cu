// FP32 variant of the logistic HMC kernel on the 5th-generation tensor cores (sm_100a), the
// "FP32 variant reported separately" of SURVEY 8(d). A CTA runs 128 chains; per 128-row tile of the
// design the two contractions of a gradient pass are computed transposed, chains on the TMEM lanes:
//   eta^T = Theta^T . X^T   (M = 128 chains, N = 128 rows, K = 56 columns)   SS form
//   G^T  += R^T . X         (M = 128 chains, N = 112 stacked columns, K = 128 rows)   TS form:
//                           R^T is written by the epilogue straight into tensor memory and read
//                           there as the A operand; it never touches shared memory.
// Operands are split exactly as x = hi + lo (hi = x rounded to TF32, lo = the FP32 remainder):
// eta^T = Th_hi.X_hi + Th_hi.X_lo + Th_lo.X_hi (3 MMAs per k-step) and
// G^T = R_hi.[X_hi | X_lo] + R_lo.[X_hi | X_lo(0..7)] (N = 112 and N = 64), FP32 accumulation in
// TMEM, flushed into FP64 per-CTA accumulators every 16 tiles. That gives FP32-class results (the
// north star's 1e-5 tolerance).
//
// Warp specialisation (544 threads): 16 epilogue warps + 1 control warp.
//  * Control thread (warp 16, lane 0): TMA bulk copies of the tile images and every tcgen05.mma.
//    Tensor-pipe order: ..., G(g-1), eta(g+1), G(g), eta(g+2), ... so the eta of the next tile
//    and the G of the previous one run while the epilogue warps work on tile g.
//  * Epilogue warp w: TMEM lane quadrant w%4 (32 chains, one per thread) x row block w/4 (32 rows).
//    Per tile: tcgen05.ld eta^T, residual r = mask(y - sigmoid(eta)) in FP32, tcgen05.st R_hi^T in
//    place over eta^T (double-buffered by tile parity), R_lo^T into its own columns once G(g-1)
//    has consumed the previous one, then one mbarrier arrive.
// TMEM (512 columns): eta/R_hi buffers 0..127 and 128..255, R_lo 256..383, G^T 384..495.
// Shared memory: Theta^T image (A of eta), eta image of X (B of eta), G image of X (B of G),
// y/keys (double-buffered); all K-major SWIZZLE_NONE canonical layouts (a tf32 MMA with an
// MN-major SWIZZLE_NONE operand returns zeros on B200: tools/probes/tf32_umma_probe.cu; the TS form
// is checked by tools/probes/tf32_ts_probe.cu).
// The chain state, integrator, energies, Metropolis test, RNG, log_pred and accumulators are FP64
// and the same as glm_kernel.cu (hmc.cpp:22-99, engine.cpp:342-381).
#include <cooperative_groups.h>
#include <math_constants.h>

#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "device_cache.hpp"
#include "device_common.cuh"
#include "tc_common.cuh"
#include "types.cuh"

namespace pcvg {

namespace {

using namespace tc;

constexpr int kC = 128;                         // chains per CTA (= UMMA M, TMEM lanes)
constexpr int kEpiWarps = 16;
constexpr int kEpiThreads = kEpiWarps * 32;     // 512
constexpr int kThreads = kEpiThreads + 32;      // + control warp
constexpr int kCtl = kEpiThreads;               // the control thread
constexpr int kOwners = kEpiThreads / kC;       // owner threads per chain (4)
constexpr int kRows = 128;                      // rows per tile (= N of eta, K of G)
constexpr int kK = 56;                          // padded design width (1 + 50 covariates + pad)
constexpr int kChunks = kK / 4;                 // 16-byte column chunks per row (14)
constexpr int kOwn = (kK + kOwners - 1) / kOwners;
constexpr int kChunkBytes = kRows * 16;         // one column chunk of the eta image (2048)
constexpr int kXImg = 2 * kChunks * kChunkBytes;  // eta image: hi + lo (57344)
constexpr int kYK = kRows * 8;                  // y (f32) + key (i32)
constexpr int kGN = 2 * kK;                     // stacked hi/lo columns (112) = N of G
constexpr int kGChunk = kGN * 16;               // one row chunk of the G image (1792)
constexpr int kGImg = (kRows / 4) * kGChunk;    // G image: [row chunk][112 stacked columns][4] (57344)
constexpr int kTileBytes = kXImg + kYK + kGImg; // per tile in HBM: eta image, y/key, G image
constexpr int kThChunk = kC * 16;               // one column chunk of the Theta^T image (2048)
constexpr int kThImg = 2 * kChunks * kThChunk;  // [hi chunks | lo chunks][chain][4] (57344)
constexpr int kFlush = 16;                      // tiles between FP32 -> FP64 flushes of G
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColE0 = 0, kColRL = 256, kColG = 384;

static_assert(kTileBytes % 16 == 0 && kXImg % 16 == 0 && kYK % 16 == 0, "bulk copy granularity");
static_assert(kThImg == kK * kC * 8, "the momentum staging [k][chain] (FP64) aliases the Theta image");
static_assert(kGN % 16 == 0 && kGN <= 128, "N of the G MMA");

struct Smem32 {
  alignas(128) unsigned char th[kThImg];
  alignas(128) unsigned char xa[kXImg];
  alignas(128) unsigned char xb[kGImg];
  alignas(128) unsigned char yk[2][kYK];
  double red[kOwners][kC];
  double pri[kOwners][kC];
  double llq[4][kC];
  int lo[kC], hi[kC], bad[kC], cur[kC];
  unsigned long long full_a, full_b, full_y[2];  // eta image, G image, y/key slots
  unsigned long long eta_bar[2], g_bar, rdy;     // eta(g) done (per buffer), G(g) done, R(g) written
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

// Instruction descriptor: kind::tf32, FP32 accumulate, M x N, both operands K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc ? 1 : 0));
}

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc ? 1 : 0));
}

__device__ __forceinline__ void mma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

// 16 consecutive 32-bit TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// 1 / (1 + 2^(-eta log2 e)) with one MUFU.EX2 and one MUFU.RCP (ftz forms: no range fix-ups);
// relative error ~2^-21. eta -> -inf gives rcp(inf) = 0, eta -> +inf gives 1, NaN propagates.
__device__ __forceinline__ float sigmoid_fast(float eta) {
  float e, s;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(eta * -1.4426950408889634f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(1.0f + e));
  return s;
}

__device__ __forceinline__ double bernoulli_logit32(double y, double x) {
  return y * x - (fmax(x, 0.0) + log1p(exp(-fabs(x))));
}

// ------------------------------------------------------------------ tile stream
// g = tiles consumed so far (over all passes); ia / ib = eta / G images issued. Load j carries
// tile j % ntiles. Every barrier completes once per tile in tile order, so the parity of tile g
// is g & 1 (per-buffer barriers eta_bar[g & 1] and full_y[g & 1]: (g >> 1) & 1).
struct Pipe32 {
  uint32_t g = 0, ia = 0, ib = 0;
  int t0 = 0;  // first row tile of this CTA (row-split clusters: rank share [t0, t0 + ntiles))
};

__device__ __forceinline__ const unsigned char* tile_src(const ModelDev& M, uint32_t j, int ntiles, int t0) {
  return M.x32 + static_cast<size_t>(t0 + static_cast<int>(j % static_cast<uint32_t>(ntiles))) * kTileBytes;
}
__device__ __forceinline__ void load_eta_image(Smem32& sm, const ModelDev& M, uint32_t j, int ntiles, int t0) {
  const unsigned char* src = tile_src(M, j, ntiles, t0);
  fence_proxy_async();
  mbar_expect_tx(&sm.full_a, kXImg);
  bulk_g2s(sm.xa, src, kXImg, &sm.full_a);
  mbar_expect_tx(&sm.full_y[j & 1], kYK);
  bulk_g2s(sm.yk[j & 1], src + kXImg, kYK, &sm.full_y[j & 1]);
}
__device__ __forceinline__ void load_g_image(Smem32& sm, const ModelDev& M, uint32_t j, int ntiles, int t0) {
  fence_proxy_async();
  mbar_expect_tx(&sm.full_b, kGImg);
  bulk_g2s(sm.xb, tile_src(M, j, ntiles, t0) + kXImg + kYK, kGImg, &sm.full_b);
}

// eta^T(g) into buffer g & 1: 7 k-steps x {hi.hi, hi.lo, lo.hi}. Descriptors advance by adding
// (byte offset >> 4) to the start-address field (no carry: every image lies below 256 KB).
__device__ __forceinline__ void issue_eta(Smem32& sm, uint32_t g) {
  constexpr uint32_t kId = idesc_tf32(128, kRows);
  const uint32_t d = sm.tmem_base + kColE0 + (g & 1u) * 128u;
  const uint64_t a0 = sdesc(sm.th, kThChunk, 128), b0 = sdesc(sm.xa, kChunkBytes, 128);
#pragma unroll
  for (int ks = 0; ks < kChunks / 2; ++ks) {
    const uint64_t ah = a0 + ((2 * ks * kThChunk) >> 4), al = a0 + (((kChunks + 2 * ks) * kThChunk) >> 4);
    const uint64_t bh = b0 + ((2 * ks * kChunkBytes) >> 4), bl = b0 + (((kChunks + 2 * ks) * kChunkBytes) >> 4);
    mma_ss(d, ah, bh, kId, ks > 0);
    mma_ss(d, ah, bl, kId, true);
    mma_ss(d, al, bh, kId, true);
  }
  mma_commit(&sm.eta_bar[g & 1]);
}

// G^T += R_hi^T(g) . [X_hi | X_lo] + R_lo^T . [X_hi | X_lo(0..7)]: 16 k-steps of 8 rows
// (measured 56 + 44 cycles per k-step: tools/probes/tf32_rate_probe.cu).
__device__ __forceinline__ void issue_g(Smem32& sm, uint32_t g, bool fresh) {
  constexpr uint32_t kIdHi = idesc_tf32(128, kGN);
  constexpr uint32_t kIdLo = idesc_tf32(128, 64);
  const uint32_t d = sm.tmem_base + kColG;
  const uint32_t rh = sm.tmem_base + kColE0 + (g & 1u) * 128u, rl = sm.tmem_base + kColRL;
  const uint64_t b0 = sdesc(sm.xb, kGChunk, 128);
#pragma unroll
  for (int ks = 0; ks < kRows / 8; ++ks) {
    const uint64_t b = b0 + ((2 * ks * kGChunk) >> 4);
    mma_ts(d, rh + 8 * ks, b, kIdHi, !(fresh && ks == 0));
    mma_ts(d, rl + 8 * ks, b, kIdLo, true);
  }
  mma_commit(&sm.g_bar);
}

#ifdef PCVG_GLM32_TRACE
// Timeline probe (tools only): clock64 stamps of CTA 0 for pass 6, printed at its end.
__device__ long long g_trace[64][10];
__device__ int g_pass;
#define TRACE(t, i)                                                         \
  do {                                                                      \
    if (blockIdx.x == 0 && g_pass == 6 && (t) < 64) g_trace[(t)][(i)] = clock64(); \
  } while (0)
#else
#define TRACE(t, i) \
  do {              \
  } while (0)
#endif

// ------------------------------------------------------------------ one gradient pass
// Accumulates G (FP64, [stacked column][chain] in gsc) over all tiles for the CTA's 128 chains
// with the parameters in the Theta image; VALUE leaves the per-chain log-likelihood in sm.llq.
// `more` = another pass follows (its first tile images may be prefetched).
template <bool VALUE>
__device__ void grad_pass32(Smem32& sm, const ModelDev& M, double* gsc, Pipe32& P, int ntiles, bool more) {
  const int tid = threadIdx.x;
  const uint32_t g0 = P.g;
  if (tid == kCtl) {
    // ---------------- control thread
    if (P.ia == g0) load_eta_image(sm, M, P.ia++, ntiles, P.t0);
    if (P.ib == g0) load_g_image(sm, M, P.ib++, ntiles, P.t0);
    mbar_wait(&sm.full_a, g0 & 1u);
    tmem_fence_after();
    issue_eta(sm, g0);
    if (ntiles > 1 || more) {
      mbar_wait(&sm.eta_bar[g0 & 1u], (g0 >> 1) & 1u);  // the eta image buffer is free
      load_eta_image(sm, M, P.ia++, ntiles, P.t0);
      if (ntiles > 1) {
        mbar_wait(&sm.full_a, (g0 + 1) & 1u);
        tmem_fence_after();
        issue_eta(sm, g0 + 1);
      }
    }
    for (int t = 0; t < ntiles; ++t) {
      const uint32_t g = g0 + t;
      mbar_wait(&sm.rdy, g & 1u);  // R^T(g) is in tensor memory
      TRACE(t, 0);
      mbar_wait(&sm.full_b, g & 1u);
      tmem_fence_after();
      issue_g(sm, g, t % kFlush == 0);
      TRACE(t, 1);
      if (t + 2 < ntiles || (t + 2 == ntiles && more)) {
        mbar_wait(&sm.eta_bar[(g + 1) & 1u], ((g + 1) >> 1) & 1u);  // eta(g+1) read the buffer
        TRACE(t, 2);
        load_eta_image(sm, M, P.ia++, ntiles, P.t0);  // y/key slot g & 1: epilogue(g) is done
        if (t + 2 < ntiles) {
          mbar_wait(&sm.full_a, (g + 2) & 1u);
          TRACE(t, 3);
          tmem_fence_after();
          issue_eta(sm, g + 2);
        }
      }
      if (t + 1 < ntiles || more) {
        mbar_wait(&sm.g_bar, g & 1u);  // G(g) read the G image buffer
        TRACE(t, 4);
        load_g_image(sm, M, P.ib++, ntiles, P.t0);
      }
    }
  } else if (tid < kEpiThreads) {
    // ---------------- epilogue warps
    const int w = tid >> 5, l = tid & 31;
    const int q = w & 3, rb = w >> 2;
    const int c = 32 * q + l;  // this thread's chain (TMEM lane)
    const uint32_t lane = static_cast<uint32_t>(32 * q) << 16;
    const int clo = sm.lo[c], chi = sm.hi[c];
    const unsigned span = static_cast<unsigned>(chi - clo);
    double llacc = 0.0;
    bool first_flush = true;
    auto flush = [&]() {  // G^T (FP32, TMEM) -> FP64 accumulators [column][chain]
      tmem_fence_after();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col0 = 32 * rb + 16 * h;
        if (col0 >= kGN) break;
        uint32_t gv[16];
        tmem_ld16(sm.tmem_base + lane + kColG + col0, gv);
        double* dst = gsc + static_cast<size_t>(col0) * kC + c;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const double v = static_cast<double>(__uint_as_float(gv[j]));
          dst[j * kC] = first_flush ? v : dst[j * kC] + v;
        }
      }
      first_flush = false;
    };
    for (int t = 0; t < ntiles; ++t) {
      const uint32_t g = g0 + t;
      if (tid == 0) TRACE(t, 5);
      mbar_wait(&sm.eta_bar[g & 1u], (g >> 1) & 1u);
      mbar_wait(&sm.full_y[g & 1u], (g >> 1) & 1u);
      if (tid == 0) TRACE(t, 6);
      tmem_fence_after();
      const uint32_t ebuf = sm.tmem_base + lane + kColE0 + (g & 1u) * 128u + 32 * rb;
      const float4* yv4 = reinterpret_cast<const float4*>(sm.yk[g & 1u]) + 8 * rb;
      const int4* kv4 = reinterpret_cast<const int4*>(sm.yk[g & 1u] + kRows * 4) + 8 * rb;
      uint32_t rlo[32];
      float ll = 0.0f;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t e[16];
        tmem_ld16(ebuf + 16 * h, e);
#pragma unroll
        for (int j4 = 0; j4 < 4; ++j4) {
          const float4 y4 = yv4[4 * h + j4];
          const int4 k4 = kv4[4 * h + j4];
          const float ys[4] = {y4.x, y4.y, y4.z, y4.w};
          const int ks[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = 4 * j4 + u;
            const float eta = __uint_as_float(e[j]);
            // padding rows (key -1) pass the fold test, but their G-image rows are zero
            const bool train = static_cast<unsigned>(ks[u] - clo) >= span;
            const float sig = sigmoid_fast(eta);
            const float r = train ? ys[u] - sig : 0.0f;
            // hi = r truncated to TF32 (exact), lo = r - hi (exact in FP32)
            const uint32_t rh = __float_as_uint(r) & 0xFFFFE000u;
            e[j] = rh;
            rlo[16 * h + j] = __float_as_uint(r - __uint_as_float(rh));
            if (VALUE) {
              const bool real = ks[u] >= 0;
              if (real && train) ll += ys[u] * eta - (fmaxf(eta, 0.0f) + log1pf(__expf(-fabsf(eta))));
              else if (real && !isfinite(eta)) ll += CUDART_NAN_F;  // 0 * non-finite test term
            }
          }
        }
        tmem_st16(ebuf + 16 * h, e);  // R_hi^T in place of eta^T
      }
      if (VALUE) llacc += static_cast<double>(ll);
      if (tid == 0) TRACE(t, 7);
      if (t > 0) {  // G(g-1) has consumed R_lo(g-1); flush it if it closed a group
        mbar_wait(&sm.g_bar, (g - 1) & 1u);
        if (tid == 0) TRACE(t, 8);
        if (t % kFlush == 0) flush();
      }
      {
        const uint32_t rl = sm.tmem_base + lane + kColRL + 32 * rb;
        uint32_t a[16], b[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          a[j] = rlo[j];
          b[j] = rlo[16 + j];
        }
        tmem_st16(rl, a);
        tmem_st16(rl + 16, b);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      tmem_fence_before();
      mbar_arrive(&sm.rdy);
      if (tid == 0) TRACE(t, 9);
    }
    mbar_wait(&sm.g_bar, (g0 + ntiles - 1) & 1u);
    flush();
    if (VALUE) sm.llq[rb][c] = llacc;
  }
  tmem_fence_before();
  __syncthreads();  // G scratch / llq complete; every buffer of the pass is released
  P.g += ntiles;
#ifdef PCVG_GLM32_TRACE
  if (blockIdx.x == 0 && tid == 0) {
    if (g_pass == 6) {
      const long long b = g_trace[0][5];
      printf("tile: ctl rdy Gissued eta(g+1)done X(g+2)landed G(g)done | epi start etaready compdone G(g-1)done arrive\n");
      for (int t = 0; t < 40 && t < ntiles; ++t)
        printf("%2d: %7lld %7lld %7lld %7lld %7lld | %7lld %7lld %7lld %7lld %7lld\n", t, g_trace[t][0] - b, g_trace[t][1] - b,
               g_trace[t][2] - b, g_trace[t][3] - b, g_trace[t][4] - b, g_trace[t][5] - b, g_trace[t][6] - b,
               g_trace[t][7] - b, g_trace[t][8] - b, g_trace[t][9] - b);
    }
    ++g_pass;
  }
#endif
}

// cs > 1: the CTAs of a cluster replicate one 128-chain tile and split its row tiles (the last
// partial wave of a launch); per pass the FP64 G partials (global scratch) and log-likelihood
// partials (DSMEM) are summed in rank order, so every rank holds identical chain state; rank 0
// owns every global write (the glm_kernel cluster scheme, glm_kernel.cu).
__global__ void __launch_bounds__(kThreads, 1) glm32_kernel(ModelDev M, ChainsDev S, RunArgs A, double* gscratch,
                                                             int cs, int tile0) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem32& sm = *reinterpret_cast<Smem32*>(smem_raw);
  const int tid = threadIdx.x;
  const int nch = S.nch;
  const int dim = M.dim;
  const size_t plane = static_cast<size_t>(dim) * nch;
  const int tile = tile0 + static_cast<int>(blockIdx.x) / cs, crank = static_cast<int>(blockIdx.x) % cs;
  const bool writer = crank == 0;
  const int ntiles_all = (M.n + kRows - 1) / kRows;
  const int rt0 = crank * ntiles_all / cs, ntiles = (crank + 1) * ntiles_all / cs - rt0;
  const bool owner = tid < kEpiThreads;
  const int oc = tid & (kC - 1), ok = tid / kC;
  const int ogc = tile * kC + oc;
  const bool ovalid = owner && ogc < nch;
  const bool is_chain = tid < kC;
  const int gc = tile * kC + tid;
  const bool cvalid = is_chain && gc < nch;
  const bool cwrite = cvalid && writer;
  double* gsc = gscratch + static_cast<size_t>(blockIdx.x) * kGN * kC;
  double* gsc0 = gscratch + static_cast<size_t>(blockIdx.x - crank) * kGN * kC;  // rank 0 of the cluster

  if (tid == 0) {
    mbar_init(&sm.full_a, 1);
    mbar_init(&sm.full_b, 1);
    mbar_init(&sm.full_y[0], 1);
    mbar_init(&sm.full_y[1], 1);
    mbar_init(&sm.eta_bar[0], 1);
    mbar_init(&sm.eta_bar[1], 1);
    mbar_init(&sm.g_bar, 1);
    mbar_init(&sm.rdy, kEpiThreads);
  }
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
      sm.cur[tid] = S.cur[gc];
      lp0 = S.lp0[gc];
      R.init(S.seed, S.rng_stream[gc], S.rng_pos[gc], S.rng_cached[gc], S.rng_has[gc] != 0);
    } else {
      sm.lo[tid] = 0;
      sm.hi[tid] = 0;
      sm.cur[tid] = 0;
    }
  }
  for (int i = tid; i < kThImg / 4; i += kThreads) reinterpret_cast<float*>(sm.th)[i] = 0.0f;
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  Pipe32 P;
  P.t0 = rt0;
  auto csync = [&]() {  // all of the cluster's G scratch / llq / chain-state writes visible
    if (cs > 1) cooperative_groups::this_cluster().sync();
    else __syncthreads();
  };

  double qown[kOwn];
  // owners publish theta (hi / lo) into the A image of eta^T: element (chain, k) at
  // (k/4) * kThChunk + chain * 16 + (k%4) * 4, lo chunks after the hi chunks
  auto put_theta = [&]() {
    if (owner) {
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        const int k = ok + kOwners * j;
        if (k < dim) {
          const float v = static_cast<float>(qown[j]);
          const float h = tf32_hi(v);
          const uint32_t off = (k >> 2) * kThChunk + oc * 16 + (k & 3) * 4;
          *reinterpret_cast<float*>(sm.th + off) = h;
          *reinterpret_cast<float*>(sm.th + kChunks * kThChunk + off) = v - h;
        }
      }
    }
    fence_proxy_async();
  };
  auto gk_of = [&](int k) {  // sum over the cluster's ranks in rank order (cs = 1: own scratch)
    double s = 0.0;
    for (int r = 0; r < cs; ++r) {
      const double* gr = gsc0 + static_cast<size_t>(r) * kGN * kC;
      s += gr[static_cast<size_t>(k) * kC + oc] + gr[static_cast<size_t>(kK + k) * kC + oc];
    }
    return s;
  };
  auto ll_of = [&](int c) {
    double s = 0.0;
    for (int r = 0; r < cs; ++r) {
      const Smem32* rm = cs > 1 ? cooperative_groups::this_cluster().map_shared_rank(&sm, r) : &sm;
      s += (rm->llq[0][c] + rm->llq[1][c]) + (rm->llq[2][c] + rm->llq[3][c]);
    }
    return s;
  };
  auto lp_from_partials = [&](int c) {
    double pr = 0.0;
#pragma unroll
    for (int o = 0; o < kOwners; ++o) pr += sm.pri[o][c];
    return ll_of(c) + pr;
  };

  if (A.mode == kModeEval) {
    const int cu = owner ? sm.cur[oc] : 0;
#pragma unroll
    for (int j = 0; j < kOwn; ++j) {
      const int k = ok + kOwners * j;
      qown[j] = (k < dim && ovalid) ? S.pos[cu * plane + static_cast<size_t>(k) * nch + ogc] : 0.0;
    }
    put_theta();
    __syncthreads();
    grad_pass32<true>(sm, M, gsc, P, ntiles, false);
    csync();
    if (owner) {
      double pr = 0.0;
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        const int k = ok + kOwners * j;
        if (k < dim) {
          if (ovalid && writer) S.grad[cu * plane + static_cast<size_t>(k) * nch + ogc] = gk_of(k) - qown[j];
          pr += -0.5 * (kLog2Pi + qown[j] * qown[j]);
        }
      }
      sm.pri[ok][oc] = pr;
    }
    __syncthreads();
    if (cwrite) {
      const double lp = lp_from_partials(tid);
      S.lp0[gc] = lp;
      if (A.out_a) A.out_a[gc] = lp;
    }
    csync();  // remote llq reads done before any rank exits
  } else {
    const double eps = M.step, half = 0.5 * M.step;
    const int n_lf = M.n_lf;
    for (int64_t it = 0; it < A.n_iters; ++it) {
      if (A.mode != kModePred) {
        // momentum refresh (chain thread, reference draw order), staged [k][chain] in the Theta
        // image (free between passes)
        double k0 = 0.0;
        double* pstage = reinterpret_cast<double*>(sm.th);
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
        if (owner) {
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
        __syncthreads();  // momentum staging read before the Theta image is overwritten
        put_theta();
        __syncthreads();
        for (int s = 0; s < n_lf; ++s) {
          const bool last = s == n_lf - 1;
          const bool more = !last || it + 1 < A.n_iters;
          if (last) grad_pass32<true>(sm, M, gsc, P, ntiles, more);
          else grad_pass32<false>(sm, M, gsc, P, ntiles, more);
          if (cs > 1) cooperative_groups::this_cluster().sync();  // every rank's G partials landed
          if (owner) {
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
                  if (ovalid && writer) {
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
          }
          csync();  // G scratch read by every owner (every rank) before the next pass rewrites it
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
          const bool bad = sm.bad[tid] != 0 || fold == M.broken_fold;
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
          if (cwrite && A.mode == kModeProbe) {
            A.out_a[gc] = h0;
            A.out_b[gc] = h1;
            A.out_flags[gc] = (accepted ? 1 : 0) | (divergent ? 2 : 0);
          }
          if (cwrite && A.mode == kModeChain) {
            const size_t row = static_cast<size_t>(it) * nch + gc;
            if (A.traj_div) A.traj_div[row] = (accepted ? 1 : 0) | (divergent ? 2 : 0);
            if (A.out_a) A.out_a[row] = h0;
            if (A.out_b) A.out_b[row] = h1;
          }
        }
        csync();  // rank 0's proposal writes and every rank's llq reads before the next transition
        if (A.mode == kModeProbe) continue;
        if (A.mode == kModeChain) {
          if (ovalid && writer && A.traj) {
            const int cu = sm.cur[oc];
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
      if (cwrite) {
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
    if (cwrite && A.mode != kModePred) {
      S.cur[gc] = static_cast<int8_t>(sm.cur[tid]);
      S.lp0[gc] = lp0;
      S.rng_pos[gc] = R.pos;
      S.rng_cached[gc] = R.cached;
      S.rng_has[gc] = R.has_cached ? 1 : 0;
      S.divergences[gc] += div_count;
      if (A.mode == kModeWarmup) S.warm_sum[gc] += warm;
    }
  }
  if (tid == kCtl) {  // no bulk copy may still be landing in shared memory at exit
    if (P.ia > P.g) {
      mbar_wait(&sm.full_a, P.g & 1u);
      mbar_wait(&sm.full_y[P.g & 1u], (P.g >> 1) & 1u);
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
// row key (int32, -1 on padding rows), then the G image [32 row chunks][112 stacked columns: hi
// 0..55, lo 56..111][4 rows].
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
        const size_t go = static_cast<size_t>(r / 4) * kGN * 4 + (r % 4);
        gi[go + static_cast<size_t>(k) * 4] = h;
        gi[go + static_cast<size_t>(kK + k) * 4] = v - h;
      }
      ys[r] = i < n ? static_cast<float>(y[i]) : 0.0f;
      ks[r] = i < n ? key[i] : -1;
    }
  }
}

// Doubles of G scratch a launch over nch chains needs at most: one [kGN][kC] block per CTA, and a
// launch has at most max(tiles, SMs) CTAs (full waves, or a tail of row-split clusters <= SMs).
size_t glm32_scratch_doubles(int nch) {
  const int tiles = (nch + kC - 1) / kC;
  return static_cast<size_t>(std::max(tiles, 256)) * kGN * kC;
}

cudaError_t launch_glm32(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st) {
  const int tiles = (S.nch + kC - 1) / kC;
  if (tiles == 0) return cudaSuccess;
  if (M.family != kLogistic || M.x32 == nullptr || M.dim > kK) return cudaErrorInvalidValue;
  {
    cudaError_t e = ensure_kernel_smem(reinterpret_cast<const void*>(glm32_kernel), sizeof(Smem32));
    if (e != cudaSuccess) return e;
  }
  const int sms = device_sm_count();
  // Wave tail: one CTA per SM, so the last partial wave of r tiles would take a full wave time. It
  // runs instead as row-split clusters of ct CTAs (same chains, summation split by rank).
  const int ntiles_rows = (M.n + kRows - 1) / kRows;
  static const bool no_split = std::getenv("PCVG_NO_TAIL_SPLIT") != nullptr;  // A/B tests only
  int r = 0, ct = 1;
  if (tiles > sms && tiles % sms != 0 && !no_split) {
    r = tiles % sms;
    while (ct < 8 && r * ct * 2 <= sms && ntiles_rows >= 4 * ct * 2) ct *= 2;
    if (ct == 1) r = 0;
  }
  if (const char* e = std::getenv("PCVG_GLM32_CS")) {  // tests / tuning: every tile row-split
    ct = std::max(1, std::atoi(e));
    r = tiles;
  }
  // one G scratch per CTA of a launch, owned by the model (its launches are stream-ordered)
  const int grid_max = std::max(tiles - r, r * ct);
  double* scratch = M.g32_scratch;
  if (scratch == nullptr || static_cast<size_t>(grid_max) * kGN * kC > glm32_scratch_doubles(S.nch))
    return cudaErrorInvalidValue;
  auto launch = [&](int tile0, int ntiles, int cs) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles * cs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sizeof(Smem32);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = cs > 1 ? 1 : 0;
    ++sampler_launch_count();
    return cudaLaunchKernelEx(&cfg, glm32_kernel, M, S, A, scratch, cs, tile0);
  };
  if (tiles - r > 0) {
    cudaError_t e = launch(0, tiles - r, 1);
    if (e != cudaSuccess) return e;
  }
  if (r > 0) return launch(tiles - r, r, ct);
  return cudaSuccess;
}

}  // namespace pcvg
