// Per-device launch facts (host side). Kernel attributes, occupancy answers and SM counts belong
// to one device context, so every cache here is keyed by the current device ordinal and guarded
// for one host thread per GPU (the multi-device context drives each device from its own thread).
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

namespace pcvg {

inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) d = 0;
  return d;
}

// Multiprocessor count of the current device (148 on B200).
inline int device_sm_count() {
  static std::mutex mu;
  static std::map<int, int> cache;
  const int d = current_device();
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(d);
  if (it != cache.end()) return it->second;
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0) v = 148;
  cache[d] = v;
  return v;
}

// Raises `fn`'s dynamic shared-memory limit to at least `bytes` on the current device (and allows
// non-portable cluster sizes when asked). Idempotent per (kernel, device).
inline cudaError_t ensure_kernel_smem(const void* fn, size_t bytes, bool nonportable_cluster = false) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  const int d = current_device();
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = done[{fn, d}];
  if (cur != 0 && bytes <= cur) return cudaSuccess;
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (e != cudaSuccess) return e;
  }
  if (nonportable_cluster) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cur = bytes < 1 ? 1 : bytes;
  return cudaSuccess;
}

// Memoised answer of `query()` for (kernel, device, key): e.g. concurrently schedulable clusters.
template <class Q>
int cached_launch_fact(const void* fn, int key, Q&& query) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int>, int> done;
  const int d = current_device();
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = done.find({fn, d, key});
    if (it != done.end()) return it->second;
  }
  const int v = query();
  std::lock_guard<std::mutex> g(mu);
  done[{fn, d, key}] = v;
  return v;
}

}  // namespace pcvg
