// Instrumentation helpers: the FFMA throughput microbenchmark that provides
// the fp32 roofline denominator, and per-kind aggregation of launch records.
#include "common.cuh"

namespace vxg {
namespace {

// 8 independent FMA chains per thread keep every FMA pipe busy; the result is
// stored conditionally so the compiler cannot drop the chains.
__global__ void __launch_bounds__(256) ffma_kernel(float* out, int iters, float seed) {
  float a0 = seed + threadIdx.x, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
  float a4 = a0 + 4.f, a5 = a0 + 5.f, a6 = a0 + 6.f, a7 = a0 + 7.f;
  const float m = 0.9999f, c = 1e-4f;
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
      a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
    }
  }
  const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1234.5f) out[threadIdx.x] = s;
}

}  // namespace

double bench_ffma(Ctx* c) {
  float* d = nullptr;
  VXG_CUDA_CHECK(cudaMalloc(&d, 1024 * sizeof(float)));
  const int blocks = c->num_sms * 8, threads = 256, iters = 4096;
  cudaEvent_t a, b;
  VXG_CUDA_CHECK(cudaEventCreate(&a));
  VXG_CUDA_CHECK(cudaEventCreate(&b));
  ffma_kernel<<<blocks, threads, 0, c->stream>>>(d, iters, 1.f);  // warm up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    VXG_CUDA_CHECK(cudaEventRecord(a, c->stream));
    ffma_kernel<<<blocks, threads, 0, c->stream>>>(d, iters, 1.f + r);
    VXG_CUDA_CHECK(cudaEventRecord(b, c->stream));
    VXG_CUDA_CHECK(cudaEventSynchronize(b));
    float ms = 0;
    VXG_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  c->counted(6);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d);
  const double flops = 2.0 * 8 * 16 * double(iters) * blocks * threads;
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace vxg
