// Microbenchmark: distributed-shared-memory store throughput inside a cluster
// (st.shared::cluster.v4, 16 B per thread, peers round-robin) against local
// st.shared.v4, and how many clusters of 2/4/8 CTAs with the contraction's
// shared-memory footprint can be co-resident on the GPU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem8 dsmem8.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int THREADS = 256, BUF = 64 * 1024, ITERS = 4096;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int REMOTE>
__global__ void st_kernel(int cs, float* sink) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  const uint32_t base = su(sm);
  float a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
  for (int it = 0; it < ITERS; ++it) {
    const uint32_t off = uint32_t(((it * THREADS + threadIdx.x) * 16) % BUF);
    if (REMOTE) {
      const uint32_t peer = (rank + 1 + (it % (cs - 1))) % cs;
      uint32_t r;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(base + off), "r"(peer));
      asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(r), "f"(a), "f"(b), "f"(c), "f"(d)
                   : "memory");
    } else {
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(base + off), "f"(a), "f"(b), "f"(c), "f"(d)
                   : "memory");
    }
    a += 1.f;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (threadIdx.x == 0 && rank == 0) sink[blockIdx.x] = reinterpret_cast<float*>(sm)[5];
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  float* sink;
  CK(cudaMalloc(&sink, 1 << 20));
  CK(cudaFuncSetAttribute(st_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(st_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(st_kernel<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int cs : {2, 4, 8}) {
    for (int smem : {BUF, 132 * 1024, 200 * 1024}) {
      cudaLaunchConfig_t cfg{};
      cfg.blockDim = dim3(THREADS);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cfg.gridDim = dim3(cs);
      int ncl = 0;
      CK(cudaOccupancyMaxActiveClusters(&ncl, st_kernel<1>, &cfg));
      printf("cluster %d smem %d KB: max active clusters %d (%d SMs of %d)\n", cs, smem / 1024, ncl, ncl * cs, nsm);
      if (smem != BUF) continue;
      for (int remote : {0, 1}) {
        cfg.gridDim = dim3(ncl * cs * 4);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(e0);
          if (remote)
            CK(cudaLaunchKernelEx(&cfg, st_kernel<1>, cs, sink));
          else
            CK(cudaLaunchKernelEx(&cfg, st_kernel<0>, cs, sink));
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = double(cfg.gridDim.x) * THREADS * ITERS * 16;
        printf("  %s stores: %.3f ms, %.1f GB/s total, %.1f B/clk/SM at 1.9 GHz\n", remote ? "DSMEM" : "local",
               ms, bytes / ms / 1e6, bytes / (ms * 1e-3) / (ncl * cs) / 1.9e9);
      }
    }
  }
  return 0;
}
