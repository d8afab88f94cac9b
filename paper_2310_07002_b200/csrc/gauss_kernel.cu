// Launchers of the row-streaming Gaussian kernels (gauss_impl.cuh): the lane-split row kernel
// (NB = 0) and the group-batched hierarchical kernel (NB > 0); the sufficient-statistics launches
// live in suff_kernel.cu so the two halves compile in parallel.
#include "gauss_impl.cuh"

namespace pcvg {

cudaError_t launch_suff_family(const ModelDev& M, const ChainsDev& S, const RunArgs& A, int T, cudaStream_t st);

namespace {

template <int FAM, int NCM, int NGM>
cudaError_t launch_family(const ModelDev& M, const ChainsDev& S, const RunArgs& A, int T,
                          cudaStream_t st) {
  const int chains_per_block = kBlock / T;
  const int grid = (S.nch + chains_per_block - 1) / chains_per_block;
  if (grid == 0) return cudaSuccess;
  ++sampler_launch_count();
  switch (T) {
    case 1: gauss_kernel<FAM, 1, NCM, NGM, 0><<<grid, kBlock, 0, st>>>(M, S, A); break;
    case 4: gauss_kernel<FAM, 4, NCM, NGM, 0><<<grid, kBlock, 0, st>>>(M, S, A); break;
    case 8: gauss_kernel<FAM, 8, NCM, NGM, 0><<<grid, kBlock, 0, st>>>(M, S, A); break;
    case 32: gauss_kernel<FAM, 32, NCM, NGM, 0><<<grid, kBlock, 0, st>>>(M, S, A); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Group-batched launch (hierarchical families with a batch layout): one warp per chain.
template <int FAM, int NCM, int NGM, int NB>
cudaError_t launch_nb(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st, int grid) {
  const size_t smem = kRing * ring_slot_bytes(M) + 16 * kRing +
                      (FAM == kRatA ? 4 : 2) * static_cast<size_t>(M.nb) * kBlock * sizeof(double);
  {
    cudaError_t e = ensure_kernel_smem(reinterpret_cast<const void*>(gauss_kernel<FAM, 32, NCM, NGM, NB>), smem);
    if (e != cudaSuccess) return e;
  }
  ++sampler_launch_count();
  gauss_kernel<FAM, 32, NCM, NGM, NB><<<grid, kBlock, smem, st>>>(M, S, A);
  return cudaGetLastError();
}

template <int FAM, int NCM, int NGM>
cudaError_t launch_batched(const ModelDev& M, const ChainsDev& S, const RunArgs& A, cudaStream_t st) {
  const int grid = (S.nch + kBlock / 32 - 1) / (kBlock / 32);
  if (grid == 0) return cudaSuccess;
  if (M.nb > kMaxBatches) return cudaErrorInvalidValue;
  if (M.nc == NCM) return launch_nb<FAM, NCM, NGM, 1 + NCM>(M, S, A, st, grid);  // exact width
  return launch_nb<FAM, NCM, NGM, 1>(M, S, A, st, grid);
}

}  // namespace

// Lanes per chain: enough threads to fill the GPU (>= ~64 resident warps worth of work per SM
// is not reachable with few chains, so few chains get whole warps), capped by the rows a lane
// would own in the smallest segment.
int gauss_lanes_per_chain(const ModelDev& M, int nch) {
  const long target_threads = static_cast<long>(device_sm_count()) * 512;
  int T = 1;
  while (T < 32 && static_cast<long>(nch) * T < target_threads) T *= 2;
  if (T == 2) T = 4;
  if (T == 16) T = 32;
  const int rows_per_group = M.J > 0 ? M.n / M.J : M.n;
  while (T > 1 && rows_per_group < 2 * T) T = T == 32 ? 8 : (T == 8 ? 4 : 1);
  return T;
}

cudaError_t launch_gauss(const ModelDev& M, const ChainsDev& S, const RunArgs& A, int T,
                         cudaStream_t st) {
  if (T == 0) {  // group-batched kernel
    if (M.nb < 1 || M.nb > kMaxBatches) return cudaErrorInvalidValue;
    if (M.family == kGrouped && M.nc <= 4) return launch_batched<kGrouped, 4, 7>(M, S, A, st);
    if (M.family == kGrouped && M.nc <= 8) return launch_batched<kGrouped, 8, 11>(M, S, A, st);
    if (M.family == kRadon) return launch_batched<kRadon, 1, 4>(M, S, A, st);
    if (M.family == kRatB) return launch_batched<kRatB, 1, 4>(M, S, A, st);
    if (M.family == kRatA) return launch_batched<kRatA, 1, 5>(M, S, A, st);
    return cudaErrorInvalidValue;
  }
  if (T < 0) return launch_suff_family(M, S, A, -T, st);  // fold sufficient statistics, -T lanes
  switch (M.family) {
    case kGrouped:
      if (M.nc > 8) return cudaErrorInvalidValue;
      return launch_family<kGrouped, 8, 11>(M, S, A, T, st);
    case kRadon:
      return launch_family<kRadon, 1, 4>(M, S, A, T, st);
    case kSeasonal:
      if (M.nc > 13) return cudaErrorInvalidValue;
      return launch_family<kSeasonal, 13, 15>(M, S, A, T, st);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace pcvg
