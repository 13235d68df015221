// Microbenchmark: the inverse tile transform's read side for candidate
// spectrum layouts.  One CTA item = one (row, map): read its whole spectrum
// (NW frequencies, complex64) once, items ordered (row, map) with map fastest,
// so CTAs of neighbouring maps run at the same time.
//   L16  line-major  [w/16][row][map][16]      128-byte reads (today's layout)
//   L4   quad        [w/4][row][map/4][4][4]   32-byte reads, 4 maps per line
//   L2   pair-major  [w/2][row][map][2]        16-byte reads, 8 maps per line
// plus a coalesced streaming read for reference.  Bytes counted = spectrum bytes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o yread yread.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ROWS = 1728, MAPS = 80, NW = 32 * 32 * 17;  // T = 32
constexpr int THREADS = 256;

__global__ void stream(const float4* __restrict__ Y, int64_t n, float* out) {
  float s = 0.f;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = __ldcs(Y + i);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 12345.f) out[0] = s;
}

// FC = frequencies per contiguous piece (16, 4, 2); MC = maps per group (1, 4, 80)
template <int FC, int MC>
__global__ void items(const float2* __restrict__ Y, int nitems, float* out) {
  constexpr int PIECE_F4 = FC / 2;  // float4s per piece
  float s = 0.f;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int map = it % MAPS, row = it / MAPS;
    const int npieces = NW / FC;
    for (int u = threadIdx.x; u < npieces * PIECE_F4; u += THREADS) {
      const int p = u / PIECE_F4, q = u % PIECE_F4;
      // [w/FC][row][map/MC][MC][FC]
      const int64_t off = ((int64_t(p) * ROWS + row) * MAPS + (map / MC) * MC + map % MC) * FC;
      const float4 v = __ldcs(reinterpret_cast<const float4*>(Y + off) + q);
      s += v.x + v.y + v.z + v.w;
    }
  }
  if (s == 12345.f) out[0] = s;
}

template <class K>
float timeit(K launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
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
  const size_t n = size_t(ROWS) * MAPS * NW;  // complex
  const size_t bytes = n * 8;
  float2* Y;
  float* out;
  CK(cudaMalloc(&Y, bytes));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(Y, 0, bytes));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto rep = [&](const char* name, float ms) { printf("%-28s %8.3f ms  %7.0f GB/s\n", name, ms, bytes / ms / 1e6); };
  // a sample of items (rows 0..191 x all maps) keeps each run short
  const int nitems = 192 * MAPS;
  const double frac = double(nitems) / (double(ROWS) * MAPS);
  auto rep_s = [&](const char* name, float ms) {
    printf("%-28s %8.3f ms  %7.0f GB/s\n", name, ms, bytes * frac / ms / 1e6);
  };
  rep("stream", timeit([&] { stream<<<sms * 8, 512>>>(reinterpret_cast<const float4*>(Y), int64_t(bytes / 16), out); }));
  for (int occ : {2, 4, 8}) {
    const int grid = sms * occ;
    printf("-- grid %d\n", grid);
    rep_s("L16 line-major 128B", timeit([&] { items<16, 1><<<grid, THREADS>>>(Y, nitems, out); }));
    rep_s("L4 quad 32B", timeit([&] { items<4, 4><<<grid, THREADS>>>(Y, nitems, out); }));
    rep_s("L2 pair-major 16B", timeit([&] { items<2, MAPS><<<grid, THREADS>>>(Y, nitems, out); }));
  }
  CK(cudaGetLastError());
  return 0;
}
