// Microbenchmark: write throughput of the contraction epilogue's store
// patterns into a line-major spectrum ([w/16][row][map][16 w] complex, 128-byte
// lines), every byte written once (1.76 GB), vs plain coalesced writes.
//   P0 coalesced          warp writes 512 contiguous bytes per instruction
//   P1 16B x-CTA          CTA tile = 128 rows x 1 pair x 80 maps, pair fastest
//                         across blockIdx (8 CTAs share each line), lane = row
//   P1m 16B x-CTA lane=map same tiles, lane = map (32 adjacent lines per instr)
//   P2 16B same-CTA       a CTA writes the 8 pairs of its (line block, rows) one
//                         after the other (line completes inside one CTA)
//   P3 32B x-CTA          tile = 2 pairs (32-byte piece, st.global.v8), 4 CTAs/line
//   P4 64B x-CTA          tile = 4 pairs, lane pairs write one 64-byte chunk
//   P5 128B x-CTA         tile = 8 pairs, 8 lanes per line (whole lines)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ystore ystore.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ROWS = 1792, CH = 80, NWB = 96, MB = 128;
constexpr int64_t LINES = int64_t(NWB) * ROWS * CH;  // 128-byte lines
constexpr int THREADS = 128;                          // 4 warps = 128 rows (one per lane)

__device__ __forceinline__ void st_v8(void* p, float4 a, float4 b) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"l"(p), "f"(a.x), "f"(a.y), "f"(a.z),
               "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
               : "memory");
}

__global__ void p0(float4* Y, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    Y[i] = make_float4(1.f, 2.f, 3.f, float(i & 7));
}

// PPT pairs per tile (1, 2, 4, 8); pieces of 16 * PPT bytes
template <int PPT, bool LANE_MAP>
__global__ void pieces(float4* Y) {
  const int ntiles = NWB * (ROWS / MB) * (8 / PPT);
  const int row = threadIdx.x;  // tile row
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int pg = t % (8 / PPT), rest = t / (8 / PPT);
    const int mb = rest % (ROWS / MB), wb = rest / (ROWS / MB);
    const int64_t rowbase = int64_t(wb) * ROWS + mb * MB;
    const float4 v = make_float4(float(row), float(t), 1.f, 2.f);
    if (PPT == 1) {
      if (!LANE_MAP) {
        for (int i = 0; i < CH; ++i) Y[((rowbase + row) * CH + i) * 8 + pg] = v;
      } else {
        // lane = map: warp w writes rows w, w+4, ... ; 32 maps per instruction
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int r = w; r < MB; r += 4)
          for (int i0 = 0; i0 < CH; i0 += 32)
            if (i0 + lane < CH) Y[((rowbase + r) * CH + i0 + lane) * 8 + pg] = v;
      }
    } else if (PPT == 2) {
      for (int i = 0; i < CH; ++i) st_v8(&Y[((rowbase + row) * CH + i) * 8 + 2 * pg], v, v);
    } else if (PPT == 4) {
      // lane pairs: (2k, 2k+1) write the two 32-byte halves of one 64-byte chunk
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
      for (int r0 = w * 32; r0 < w * 32 + 32; r0 += 16)
        for (int i = 0; i < CH; ++i) {
          const int r = r0 + (lane >> 1);
          st_v8(&Y[((rowbase + r) * CH + i) * 8 + 4 * pg + 2 * (lane & 1)], v, v);
        }
    } else {
      // 8 lanes per 128-byte line: a warp instruction writes 4 whole lines
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
      for (int r = w * 32; r < w * 32 + 32; ++r)
        for (int i0 = 0; i0 < CH; i0 += 4)
          Y[((rowbase + r) * CH + i0 + (lane >> 3)) * 8 + (lane & 7)] = v;
    }
  }
}

// quad layout [w/4][row][map/4][4 maps][4 w]: tile = 128 rows x 1 pair x 80
// maps, lane = map: a warp instruction writes 32 pieces at 32-byte stride
// (8 lines, half of each; the CTA of the other pair writes the other half)
__global__ void p6(float4* Y) {
  const int ntiles = NWB * 8 * (ROWS / MB);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int pip = t & 7, rest = t >> 3;
    const int mb = rest % (ROWS / MB), wb = rest / (ROWS / MB);
    const int pair = wb * 8 + pip, pq = pair >> 1, half = pair & 1;
    const float4 v = make_float4(float(lane), float(t), 1.f, 2.f);
    for (int r = w; r < MB; r += 4)
      for (int i0 = 0; i0 < CH; i0 += 32)
        if (i0 + lane < CH) Y[((int64_t(pq) * ROWS + mb * MB + r) * CH + i0 + lane) * 2 + half] = v;
  }
}

// 16-byte pieces, one CTA writes all 8 pairs of its (line block, row block)
__global__ void p2(float4* Y) {
  const int ntiles = NWB * (ROWS / MB);
  const int row = threadIdx.x;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int mb = t % (ROWS / MB), wb = t / (ROWS / MB);
    const int64_t rowbase = int64_t(wb) * ROWS + mb * MB;
    const float4 v = make_float4(float(row), float(t), 1.f, 2.f);
    for (int pg = 0; pg < 8; ++pg)
      for (int i = 0; i < CH; ++i) Y[((rowbase + row) * CH + i) * 8 + pg] = v;
  }
}

template <class K>
float timeit(K launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  float4* Y;
  const size_t bytes = size_t(LINES) * 128;
  CK(cudaMalloc(&Y, bytes));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto rep = [&](const char* name, float ms) { printf("%-28s %8.3f ms  %7.0f GB/s\n", name, ms, bytes / ms / 1e6); };
  for (int occ : {1, 2, 4}) {
    const int grid = sms * occ;
    printf("-- grid %d (%d CTAs/SM of 128 threads)\n", grid, occ);
    rep("P0 coalesced", timeit([&] { p0<<<grid, 512>>>(Y, int64_t(bytes / 16)); }));
    rep("P1 16B x-CTA lane=row", timeit([&] { pieces<1, false><<<grid, THREADS>>>(Y); }));
    rep("P1m 16B x-CTA lane=map", timeit([&] { pieces<1, true><<<grid, THREADS>>>(Y); }));
    rep("P2 16B same-CTA", timeit([&] { p2<<<grid, THREADS>>>(Y); }));
    rep("P6 quad lane=map", timeit([&] { p6<<<grid, THREADS>>>(Y); }));
    rep("P3 32B x-CTA", timeit([&] { pieces<2, false><<<grid, THREADS>>>(Y); }));
    rep("P4 64B x-CTA", timeit([&] { pieces<4, false><<<grid, THREADS>>>(Y); }));
    rep("P5 128B lines", timeit([&] { pieces<8, false><<<grid, THREADS>>>(Y); }));
  }
  CK(cudaGetLastError());
  return 0;
}
