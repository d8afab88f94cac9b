// Throughput of tcgen05 kind::tf32 MMA shapes used by glm32_kernel.cu on B200: one thread per CTA
// issues a tight, fully unrolled series, one CTA per SM, commit + wait only at the end; prints
// SM cycles per MMA. SS = both operands in shared memory (SWIZZLE_NONE K-major), TS = A in TMEM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  const uint64_t a = (saddr(p) >> 4) & 0x3FFFu;
  return a | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) | (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, int acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void wait(unsigned long long* bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(saddr(bar)), "r"(ph) : "memory");
}

// TS: 0 = SS, 1 = TS. ALT: alternate two accumulators.
template <int TS, int N, int ALT>
__global__ void rate(int reps, long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* a_s = sm;
  unsigned char* b_s = sm + 65536;
  __shared__ uint32_t tbase;
  __shared__ unsigned long long bar;
  for (int i = threadIdx.x; i < 2 * 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i % 7);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint64_t da = sdesc(a_s, 2048, 128), db = sdesc(b_s, 2048, 128);
    constexpr uint32_t id = idesc_tf32(128, N);
    const uint32_t d0 = tbase + 256, d1 = tbase + (N <= 128 ? 384 : 256);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        const uint32_t d = (ALT && (ks & 1)) ? d1 : d0;
        const uint64_t b = db + ((2 * (ks % 8) * 2048) >> 4);
        if (TS) mma_ts(d, tbase + 8 * ks, b, id, 1);
        else mma_ss(d, da + ((2 * (ks % 8) * 2048) >> 4), b, id, 1);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)) : "memory");
    wait(&bar, 0);
    out[blockIdx.x] = (clock64() - t0) / (16 * reps);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
}

template <int TS, int N, int ALT>
void run() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(rate<TS, N, ALT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536);
  rate<TS, N, ALT><<<148, 128, 2 * 65536>>>(256, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%s M=128 N=%3d K=8 %s: %s  %lld cycles/MMA  (%.0f flop/cycle/SM)\n", TS ? "TS" : "SS", N, ALT ? "2 accumulators" : "1 accumulator ",
         cudaGetErrorString(e), mx, 2.0 * 128 * N * 8 / mx);
  cudaFree(d);
}

int main() {
  run<0, 64, 0>();
  run<0, 112, 0>();
  run<0, 128, 0>();
  run<0, 256, 0>();
  run<1, 64, 0>();
  run<1, 112, 0>();
  run<1, 128, 0>();
  run<1, 256, 0>();
  run<0, 128, 1>();
  run<1, 112, 1>();
  return 0;
}
