// DMMA (mma.sync m8n8k4 f64) dependent-chain latency and throughput vs independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void chain_kernel(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int t = 0; t < CH; ++t) c[t][0] = c[t][1] = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < CH; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int t = 0; t < CH; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
void run(double* out, long long* cyc, int warps_per_sm, int sms) {
  const int iters = 4000;
  chain_kernel<CH><<<sms, 32 * warps_per_sm>>>(out, 10, cyc);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  chain_kernel<CH><<<sms, 32 * warps_per_sm>>>(out, iters, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("chains/warp %2d warps/SM %2d: %.2f cyc per DMMA per warp, %.1f TF/s\n", CH, warps_per_sm,
         (double)c / (iters * CH), 2.0 * 256 * CH * iters * 32.0 / 32 * warps_per_sm * sms / (ms * 1e-3) / 1e12);
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1>(out, cyc, 1, sms); run<2>(out, cyc, 1, sms); run<4>(out, cyc, 1, sms); run<8>(out, cyc, 1, sms);
  run<1>(out, cyc, 4, sms); run<2>(out, cyc, 4, sms); run<4>(out, cyc, 4, sms); run<8>(out, cyc, 4, sms);
  run<2>(out, cyc, 8, sms); run<4>(out, cyc, 8, sms); run<8>(out, cyc, 8, sms);
  run<2>(out, cyc, 16, sms); run<4>(out, cyc, 16, sms);
  return 0;
}
