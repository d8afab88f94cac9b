// FP64 roofline probe for B200 (sm_100a): DFMA pipe and DMMA (mma.sync m8n8k4 f64).
// MEASURED_PEAKS.json carries only HBM and bf16 figures; the PCV sampler is FP64,
// so its roofline denominator is measured here. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <int TILES>
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[TILES][2];
#pragma unroll
  for (int t = 0; t < TILES; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}

// Warps 0..3 of each block run DMMA, warps 4..7 run DFMA: if the two share the FP64 datapath the
// combined rate stays at the single-pipe peak.
__global__ void mixed_kernel(double* out, int iters, int dfma_warps) {
  const int w = threadIdx.x >> 5;
  if (w < 8 - dfma_warps) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    if (s == 12345.678) out[0] = s;
  } else {
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters * 8; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], 1.0000001, 1e-9);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.678) out[0] = s;
  }
}

__global__ void dexp_kernel(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = -1.0 - 1e-3 * i - threadIdx.x * 1e-6;
  double s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { s += exp(x[i]); x[i] -= 1e-9; }
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out;
  CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  // DFMA: 8 independent chains per thread, 256 threads per block, 8 blocks/SM.
  for (int bps : {4, 8}) {
    const int iters = 20000, threads = 256, blocks = sms * bps;
    dfma_kernel<8><<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8 * iters * (double)threads * blocks;
    printf(", \"dfma_tflops_bps%d\": %.3f", bps, flops / (best * 1e-3) / 1e12);
  }
  for (int bps : {2, 4, 8}) {
    const int iters = 20000, threads = 128, blocks = sms * bps;
    dmma_kernel<8><<<blocks, threads>>>(out, 100);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      dmma_kernel<8><<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * blocks;
    printf(", \"dmma_tflops_bps%d\": %.3f", bps, flops / (best * 1e-3) / 1e12);
  }
  {
    const int iters = 2000, threads = 256, blocks = sms * 8;
    dexp_kernel<<<blocks, threads>>>(out, 10);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dexp_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"dexp_gops\": %.3f", 8.0 * iters * threads * (double)blocks / (ms * 1e-3) / 1e9);
  }
  for (int dw : {0, 2, 4, 8}) {
    const int iters = 4000, threads = 256, blocks = sms * 2;
    mixed_kernel<<<blocks, threads>>>(out, 10, dw);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    mixed_kernel<<<blocks, threads>>>(out, iters, dw);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // DMMA warp: 8*iters DMMA x 256 FMA; DFMA warp: 64*iters DFMA x 32 FMA (equal FMA count)
    const double fma_per_warp = 8.0 * iters * 256;
    printf(", \"mixed_dfma_warps%d_ms\": %.3f, \"mixed_dfma_warps%d_tflops\": %.3f", dw, ms, dw,
           2.0 * fma_per_warp * 8 * blocks / (ms * 1e-3) / 1e12);
  }
  printf("}\n");
  return 0;
}
