// Probe of the tcgen05 kind::tf32 operand layouts used by glm32_kernel.cu: one M=128 MMA with
// (a) K-major A / K-major B (the eta contraction) and (b) MN-major A / K-major B (the G
// contraction), SWIZZLE_NONE descriptors, checked against a CPU product. Result on B200: K-major
// exact; MN-major A (element (m,k) at (m/4)*SBO + (k%8)*16 + (m%4)*4) returned all zeros, so
// glm32_kernel.cu uses K-major images for both operands.
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
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
// A: M=128 x K=8 ; B: K=8 x N ; D: 128 x N fp32. Smem images: A, B as floats at given layouts.
template <int N>
__global__ void probe(const float* aimg, int abytes, const float* bimg, int bbytes, uint32_t albo, uint32_t asbo,
                      uint32_t blbo, uint32_t bsbo, int a_mn, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ unsigned long long bar;
  float* A = reinterpret_cast<float*>(sm);
  float* B = reinterpret_cast<float*>(sm + abytes);
  for (int i = threadIdx.x; i < abytes / 4; i += blockDim.x) A[i] = aimg[i];
  for (int i = threadIdx.x; i < bbytes / 4; i += blockDim.x) B[i] = bimg[i];
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tbase)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint64_t da = sdesc(A, albo, asbo), db = sdesc(B, blbo, bsbo);
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tbase),
                 "l"(da), "l"(db), "r"(idesc_tf32(128, N, a_mn, 0)));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(saddr(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tbase + ((32u * w) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[(32 * w + l) * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(128));
}

int main() {
  const int M = 128, K = 8, N = 64;
  std::vector<float> a(M * K), b(K * N);
  for (int i = 0; i < M * K; ++i) a[i] = float((i * 7) % 13) - 6.0f;
  for (int i = 0; i < K * N; ++i) b[i] = float((i * 5) % 11) - 5.0f;
  std::vector<float> ref(M * N, 0.0f);
  for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) ref[m * N + n] += a[m * K + k] * b[k * N + n];
  // B K-major: element (n, k) at (k/4)*(N*16) + n*16 + (k%4)*4 -> LBO = N*16, SBO = 128
  std::vector<float> bimg(2 * N * 4);
  for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) bimg[((k / 4) * N * 16 + n * 16 + (k % 4) * 4) / 4] = b[k * N + n];
  // (a) A K-major: element (m, k) at (k/4)*(M*16) + m*16 + (k%4)*4 -> LBO = M*16, SBO = 128
  std::vector<float> aimgK(2 * M * 4);
  for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) aimgK[((k / 4) * M * 16 + m * 16 + (k % 4) * 4) / 4] = a[m * K + k];
  // (b) A MN-major: element (m, k) at (m/4)*SBO + (k%8)*16 + (k/8)*LBO + (m%4)*4, SBO = K*16 = 128 (K=8)
  std::vector<float> aimgMN(M * K);
  const int sboMN = 8 * 16;
  for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) aimgMN[((m / 4) * sboMN + (k % 8) * 16 + (m % 4) * 4) / 4] = a[m * K + k];
  float *da, *db, *dout;
  cudaMalloc(&da, 4 * M * K); cudaMalloc(&db, 4 * K * N); cudaMalloc(&dout, 4 * M * N);
  cudaMemcpy(db, bimg.data(), 4 * K * N, cudaMemcpyHostToDevice);
  std::vector<float> out(M * N);
  for (int variant = 0; variant < 3; ++variant) {
    const bool mn = variant >= 1;
    cudaMemcpy(da, (mn ? aimgMN : aimgK).data(), 4 * M * K, cudaMemcpyHostToDevice);
    uint32_t albo = mn ? 128 : M * 16, asbo = mn ? sboMN : 128;
    if (variant == 2) { uint32_t t = albo; albo = asbo; asbo = t; }  // swapped roles
    cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * (M * K + K * N));
    probe<N><<<1, 128, 4 * (M * K + K * N)>>>(da, 4 * M * K, db, 4 * K * N, albo, asbo, N * 16, 128, mn ? 1 : 0, dout);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(out.data(), dout, 4 * M * N, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int i = 0; i < M * N; ++i) { err = fmax(err, fabs(out[i] - ref[i])); mx = fmax(mx, fabs(ref[i])); }
    printf("variant %d (%s A, lbo %u sbo %u): %s max|err| %.3g (max|ref| %.3g) out[0..3] %g %g %g %g ref %g %g %g %g\n",
           variant, mn ? "MN-major" : "K-major", albo, asbo, cudaGetErrorString(e), err, mx, out[0], out[1], out[2], out[3],
           ref[0], ref[1], ref[2], ref[3]);
  }
  return 0;
}
