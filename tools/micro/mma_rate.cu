// Microbenchmark: cycles per tcgen05.mma kind::tf32 (M = 128, K = 8) as a
// function of N, A from shared memory or tensor memory, 1 CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return uint64_t((a >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (uint64_t(1) << 46);
}
template <int N, int M = 128>
__device__ __forceinline__ constexpr uint32_t idesc() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

template <int N, bool TA, int M = 128, bool VARY = false, bool RAND = false, int GROUP = 0>
__global__ void k(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t gbar[2];
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&gbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&gbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) {
    // RAND: tf32-ish random operands (power / data dependence), else zeros
    uint32_t h = (uint32_t(i) * 2654435761u) ^ (blockIdx.x * 97u);
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    reinterpret_cast<float*>(sm)[i] = RAND ? (float(h & 0xFFFF) / 65536.f - 0.5f) : 0.f;
  }
  if (RAND && threadIdx.x < 32 * 4 && false) {}
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint64_t a = desc(su(sm));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = M == 64 ? tm + ((i & 1) << 20) : tm + (VARY ? (i & 3) * 80 : (i & 1) * 128);
      const uint64_t b = desc(su(sm + 16384 + (VARY ? (i & 7) * 2560 : 0)));
      if (TA)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5,%5,%5,%5}, p;\n}\n"
                     ::"r"(d), "r"(tm + 384 + (VARY ? (i & 7) * 8 : 0)), "l"(b), "r"(idesc<N, M>()), "r"(i > 1 ? 1 : 0), "r"(0));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5,%5,%5,%5}, p;\n}\n"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc<N, M>()), "r"(i > 1 ? 1 : 0), "r"(0));
      // GROUP: every 12 MMAs, GROUP commits (to mbarriers nobody waits on) + a fence
      // GROUP = commits*10 + fence (1) ; group of 12 MMAs (GS 24 when GROUP >= 100)
      if (GROUP && i % (GROUP >= 100 ? 24 : 12) == (GROUP >= 100 ? 23 : 11)) {
        for (int c = 0; c < (GROUP % 100) / 10; ++c)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su(&gbar[c & 1])));
        if (GROUP % 10) asm volatile("tcgen05.fence::after_thread_sync;\n");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su(&bar)));
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(su(&bar)));
    out[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
}

template <int N, bool TA, int M = 128, bool VARY = false, bool RAND = false, int GROUP = 0>
void run(long long* d) {
  cudaFuncSetAttribute(k<N, TA, M, VARY, RAND, GROUP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 19992;
  k<N, TA, M, VARY, RAND, GROUP><<<148, 128, 65536>>>(iters, d);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += h[i] / 148.0;
  printf("group=%d rand=%d vary=%d M=%d N=%3d A=%s: %.1f cycles/MMA  (%.0f MAC/clk/SM)  %s\n", GROUP, int(RAND), int(VARY), M, N, TA ? "tmem" : "smem", m / iters,
         double(M) * N * 8 * iters / m, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<80, true>(d); run<80, true, 128, true>(d); run<80, false, 128, true>(d);
  run<160, true, 128, true>(d); run<80, false, 64, true>(d);
  run<80, true, 128, true, true>(d); run<80, false, 128, true, true>(d); run<160, true, 128, true, true>(d);
  run<128, true, 128, true, true>(d); run<64, true, 128, true, true>(d);
  run<80, true, 128, true, false, 1>(d); run<80, true, 128, true, false, 10>(d); run<80, true, 128, true, false, 20>(d);
  run<80, true, 128, true, false, 11>(d); run<80, true, 128, true, false, 21>(d); run<80, true, 128, true, false, 121>(d);
  return 0;
}
