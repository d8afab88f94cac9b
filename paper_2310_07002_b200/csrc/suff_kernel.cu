// Launchers of the sufficient-statistics kernel (gauss_impl.cuh, suff_pass).
#include <cstdlib>

#include "gauss_impl.cuh"

namespace pcvg {

namespace {

// NB = -1: sufficient statistics at full registers; NB = -2 (one lane per chain, many chains):
// capped at 128 registers for 4 CTAs/SM - its spills cost latency that only pays back when the
// extra warps have chains to run (cfg5 +9%, cfg1 / cfg4 -20%).
template <int FAM, int NCM, int NGM, int T, int NB = -1>
cudaError_t launch_suff_t(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st) {
  const int grid = (S.nch + kBlock / T - 1) / (kBlock / T);
  if (grid == 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(suff_slots(M, T)) * suff_slot_arrays(M) * kBlock * sizeof(double);
  {
    cudaError_t e = ensure_kernel_smem(reinterpret_cast<const void*>(gauss_kernel<FAM, T, NCM, NGM, NB>), smem);
    if (e != cudaSuccess) return e;
  }
  ++sampler_launch_count();
  gauss_kernel<FAM, T, NCM, NGM, NB><<<grid, kBlock, smem, st>>>(M, S, A);
  return cudaGetLastError();
}

template <int FAM, int NCM, int NGM>
cudaError_t launch_suff(const ModelDev& M, const ChainsDev& S, const RunArgs& A, int T, cudaStream_t st) {
  switch (T) {
    case 1:
      if (S.nch >= device_sm_count() * 2 * kBlock * 2) return launch_suff_t<FAM, NCM, NGM, 1, -2>(M, S, A, st);
      return launch_suff_t<FAM, NCM, NGM, 1>(M, S, A, st);
    case 4: return launch_suff_t<FAM, NCM, NGM, 4>(M, S, A, st);
    case 8: return launch_suff_t<FAM, NCM, NGM, 8>(M, S, A, st);
    case 32: return launch_suff_t<FAM, NCM, NGM, 32>(M, S, A, st);
    default: return cudaErrorInvalidValue;
  }
}

// One lane per chain only (the many-chain throughput case, cfg1 / cfg5 linear regression with
// P = 5): a narrower width class keeps the unrolled Gram product and parameter loops at the
// model's size (21 instead of 45 Gram entries, 8 instead of 11 global parameters).
template <int FAM, int NCM, int NGM>
cudaError_t launch_suff1(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st) {
  if (S.nch >= device_sm_count() * 2 * kBlock * 2) return launch_suff_t<FAM, NCM, NGM, 1, -2>(M, S, A, st);
  return launch_suff_t<FAM, NCM, NGM, 1>(M, S, A, st);
}

}  // namespace

// Lanes per chain of the sufficient-statistics kernel: enough threads to fill the GPU, at most
// what the Gram entries / groups can use.
int suff_lanes_per_chain(const ModelDev& M, int nch) {
  if (const char* env = std::getenv("PCVG_SUFF_LANES")) return std::atoi(env);  // tuning only
  // Split lanes only pay for many groups: the per-pass partial sums cost (nc + 5) butterfly
  // reductions, more than a lane saves on a d(d+1)/2 Gram product (measured: cfg1 / cfg4 are
  // fastest at one lane, cfg3's 400 groups at 32, profiles/r01_suff_lanes.txt).
  if (M.J < 64) return 1;
  const long target_threads = static_cast<long>(device_sm_count()) * 512;
  int T = 1;
  while (T < 32 && static_cast<long>(nch) * T < target_threads) T *= 2;
  if (T == 2) T = 4;
  if (T == 16) T = 32;
  return T;
}

cudaError_t launch_suff_family(const ModelDev& M, const ChainsDev& S, const RunArgs& A, int T, cudaStream_t st) {
  if (!M.suff) return cudaErrorInvalidValue;
  switch (M.family) {
    case kGrouped:
      if (M.nc > 8) return cudaErrorInvalidValue;
      if (M.nc <= 5 && T == 1) return launch_suff1<kGrouped, 5, 8>(M, S, A, st);
      return launch_suff<kGrouped, 8, 11>(M, S, A, T, st);
    case kRadon:
      return launch_suff<kRadon, 1, 4>(M, S, A, T, st);
    case kRatB:  // rat growth with a shared slope: m = alpha_g + beta t (rat_growth.cpp:148-172)
      return launch_suff<kRatB, 1, 4>(M, S, A, T, st);
    case kRatA:  // per-subject slopes: per-subject (y, t) Gram (rat_growth.cpp:117-147)
      return launch_suff<kRatA, 1, 5>(M, S, A, T, st);
    case kSeasonal:
      if (M.nc > 13) return cudaErrorInvalidValue;
      return launch_suff<kSeasonal, 13, 15>(M, S, A, T, st);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace pcvg
