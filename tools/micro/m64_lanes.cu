// Where does a tcgen05.mma M=64 (cta_group::1) accumulator land in TMEM, and
// can a second one live at a lane offset?  A = B = 1 (tf32), K = 8 -> D = 8.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return uint64_t((a >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (uint64_t(1) << 46);
}
__global__ void k(int lane_off, int m, float* out) {
  __shared__ __align__(1024) float A[128 * 8], B[16 * 8];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) A[i] = 1.f;
  for (int i = threadIdx.x; i < 16 * 8; i += blockDim.x) B[i] = 1.f;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = slot;
  // zero the accumulator area first via tcgen05.st (all 128 lanes x 16 cols)
  {
    const int w = threadIdx.x >> 5;
    uint32_t z = 0;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n"
                 ::"r"(tm + (uint32_t(w * 32) << 16)), "r"(z));
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (threadIdx.x == 0) {
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(16 >> 3) << 17) | (uint32_t(m >> 4) << 24);
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5,%5,%5,%5}, p;\n}\n"
                 ::"r"(tm + (uint32_t(lane_off) << 16)), "l"(desc(su(A))), "l"(desc(su(B))), "r"(id), "r"(0), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su(&bar)));
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(su(&bar)));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  uint32_t v[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(tm + (uint32_t(w * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n");
  for (int c = 0; c < 16; ++c) out[(w * 32 + l) * 16 + c] = __uint_as_float(v[c]);
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tm));
}
int main(int argc, char** argv) {
  float* d; cudaMalloc(&d, 128 * 16 * 4);
  float h[128 * 16];
  const int m = atoi(argv[1]), off = atoi(argv[2]);
  {
      cudaMemset(d, 0, sizeof(h));
      k<<<1, 128>>>(off, m, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("M=%d lane_off=%2d (%s): lanes with D=8 in col 0..15: ", m, off, cudaGetErrorString(e));
      int start = -1;
      for (int r = 0; r <= 128; ++r) {
        bool on = r < 128 && h[r * 16] == 8.f && h[r * 16 + 15] == 8.f;
        if (on && start < 0) start = r;
        if (!on && start >= 0) { printf("[%d,%d) ", start, r); start = -1; }
      }
      printf("\n");
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
