// Microbenchmark: throughput of 16-byte-piece gathers/scatters (one frequency
// pair of a 128-byte spectrum line, the tcgen05 contraction's access pattern)
// via (a) LDGSTS 16 B, (b) TMA 5D tensor loads, (c) TMA 5D tensor stores.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma16 tma16.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ROWS = 1792, CH = 80, NWB = 96, MB = 128, KC = 8;
constexpr int SLOTS = 4, BOX = MB * KC * 16;  // 16 KB

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ldgsts_kernel(const float4* X, int ntiles) {
  extern __shared__ __align__(128) uint8_t sm[];
  int lane = threadIdx.x;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int pip = t & 7, rest = t >> 3, mb = rest % (ROWS / MB), wb = rest / (ROWS / MB);
    for (int kc = 0; kc < CH / KC; ++kc) {
      uint8_t* slot = sm + ((t * 10 + kc) % SLOTS) * BOX;
      for (int u = lane; u < MB * KC; u += 32) {
        int row = u >> 3, jj = u & 7;
        const float4* src = X + ((int64_t(wb) * ROWS + mb * MB + row) * CH + kc * KC + jj) * 8 + pip;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su(slot + u * 16)), "l"(src));
      }
      asm volatile("cp.async.commit_group;\n");
      asm volatile("cp.async.wait_group 2;\n");
    }
  }
  asm volatile("cp.async.wait_group 0;\n");
}

__global__ void tma_load_kernel(const __grid_constant__ CUtensorMap tm, int ntiles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SLOTS * BOX);
  if (threadIdx.x == 0) {
    for (int s = 0; s < SLOTS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int g = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int pip = t & 7, rest = t >> 3, mb = rest % (ROWS / MB), wb = rest / (ROWS / MB);
    for (int kc = 0; kc < CH / KC; ++kc, ++g) {
      int s = g % SLOTS;
      if (g >= SLOTS) {
        uint32_t par = ((g / SLOTS) - 1) & 1;
        asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(su(&bar[s])), "r"(par));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su(&bar[s])), "r"(BOX));
      asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
                   ::"r"(su(sm + s * BOX)), "l"(&tm), "r"(0), "r"(pip), "r"(kc * KC), "r"(mb * MB), "r"(wb), "r"(su(&bar[s])) : "memory");
    }
  }
  for (int k = 0; k < SLOTS && k < g; ++k) {
    int gg = g - 1 - k, s = gg % SLOTS;
    uint32_t par = (gg / SLOTS) & 1;
    asm volatile("{\n.reg .pred P;\nW2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W2;\n}\n" ::"r"(su(&bar[s])), "r"(par));
  }
}

__global__ void tma_store_kernel(const __grid_constant__ CUtensorMap tm, int ntiles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  if (threadIdx.x != 0) return;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int pip = t & 7, rest = t >> 3, mb = rest % (ROWS / MB), wb = rest / (ROWS / MB);
    for (int kc = 0; kc < CH / KC; ++kc) {
      asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n"
                   ::"l"(&tm), "r"(0), "r"(pip), "r"(kc * KC), "r"(mb * MB), "r"(wb), "r"(su(sm + (kc % SLOTS) * BOX)) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n");
      asm volatile("cp.async.bulk.wait_group.read 2;\n");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;\n");
}

int main() {
  size_t bytes = size_t(NWB) * ROWS * CH * 128;
  float4* X;
  CK(cudaMalloc(&X, bytes));
  CK(cudaMemset(X, 0, bytes));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t dims[5] = {4, 8, CH, ROWS, NWB};
  cuuint64_t strides[4] = {16, 128, uint64_t(CH) * 128, uint64_t(ROWS) * CH * 128};
  cuuint32_t box[5] = {4, 1, KC, MB, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return 1; }
  int ntiles = NWB * (ROWS / MB) * 8;
  int smem = SLOTS * BOX + 64;
  CK(cudaFuncSetAttribute(ldgsts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(tma_load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(tma_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int which = 0; which < 3; ++which) {
    for (int blocks : {148, 296}) {
      float best = 1e9;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        if (which == 0) ldgsts_kernel<<<blocks, 32, smem>>>(X, ntiles);
        if (which == 1) tma_load_kernel<<<blocks, 32, smem>>>(tm, ntiles);
        if (which == 2) tma_store_kernel<<<blocks, 32, smem>>>(tm, ntiles);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep) best = ms < best ? ms : best;
      }
      CK(cudaGetLastError());
      printf("%-10s blocks %d: %.3f ms  %.0f GB/s useful (16-byte pieces)\n",
             which == 0 ? "LDGSTS16" : which == 1 ? "TMA-load" : "TMA-store", blocks, best, bytes / best / 1e6);
    }
  }
  return 0;
}
