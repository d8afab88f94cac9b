// Probe of the tcgen05 kind::tf32 "TS" form used by glm32_kernel.cu: A (M=128 x K=8) in tensor
// memory written by tcgen05.st (lane = m, one 32-bit column per k), B (K=8 x N) K-major in shared
// memory (SWIZZLE_NONE), N = 112 and N = 64, D in tensor memory; checked against a CPU product.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  const uint64_t a = (saddr(p) >> 4) & 0x3FFFu;
  return a | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) | (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
template <int N>
__global__ void probe(const float* a, const float* bimg, float* out, int accumulate_twice) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ unsigned long long bar;
  float* B = reinterpret_cast<float*>(sm);
  for (int i = threadIdx.x; i < 8 * N; i += blockDim.x) B[i] = bimg[i];
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, m = 32 * w + l;
  // A row m -> TMEM lane m, columns 128..135
  {
    uint32_t r[8];
    for (int k = 0; k < 8; ++k) r[k] = __float_as_uint(a[m * 8 + k]);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tbase + ((32u * w) << 16) + 128),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint64_t db = sdesc(B, N * 16, 128);
    for (int rep = 0; rep <= accumulate_twice; ++rep)
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tbase),
                   "r"(tbase + 128), "l"(db), "r"(idesc_tf32(128, N)), "r"(rep));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(saddr(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tbase + ((32u * w) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[m * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
}

template <int N>
void run(int twice) {
  const int M = 128, K = 8;
  std::vector<float> a(M * K), b(K * N);
  for (int i = 0; i < M * K; ++i) a[i] = float((i * 7) % 13) - 6.0f;
  for (int i = 0; i < K * N; ++i) b[i] = float((i * 5) % 11) - 5.0f;
  std::vector<float> ref(M * N, 0.0f);
  for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) ref[m * N + n] += (twice + 1) * a[m * K + k] * b[k * N + n];
  std::vector<float> bimg(K * N);  // (n, k) at (k/4)*(N*16) + n*16 + (k%4)*4
  for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) bimg[((k / 4) * N * 16 + n * 16 + (k % 4) * 4) / 4] = b[k * N + n];
  float *da, *db, *dout;
  cudaMalloc(&da, 4 * M * K); cudaMalloc(&db, 4 * K * N); cudaMalloc(&dout, 4 * M * N);
  cudaMemcpy(da, a.data(), 4 * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(db, bimg.data(), 4 * K * N, cudaMemcpyHostToDevice);
  probe<N><<<1, 128, 4 * K * N>>>(da, db, dout, twice);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> out(M * N);
  cudaMemcpy(out.data(), dout, 4 * M * N, cudaMemcpyDeviceToHost);
  double err = 0, mx = 0;
  for (int i = 0; i < M * N; ++i) { err = fmax(err, fabs(out[i] - ref[i])); mx = fmax(mx, fabs(ref[i])); }
  printf("TS N=%d accumulate=%d: %s max|err| %.3g (max|ref| %.3g) out[0..3] %g %g %g %g ref %g %g %g %g\n", N, twice,
         cudaGetErrorString(e), err, mx, out[0], out[1], out[2], out[3], ref[0], ref[1], ref[2], ref[3]);
}

int main() {
  run<112>(0);
  run<64>(0);
  run<112>(1);
  return 0;
}
