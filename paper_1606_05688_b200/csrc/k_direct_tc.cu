// K5 on the tensor cores for single-input-map layers (the first layer of every
// bundled net): conv_direct / accumulate_valid_conv (proj/include/voxin/
// layers.hpp:120-192) with f = 1 as an implicit GEMM
//   out[j](x, y, z0 + m) = act(bias[j] + sum_q A[m][q] W[j][q]),
//   A[m][q] = in(x + kx-1-qx, y + ky-1-qy, z0 + m + kz-1-qz)
// M = 128 z-consecutive output voxels of one (x, y) row, N = the channel block
// (16..80 maps), K = k^3 taps padded to a multiple of 8 (k <= 4), tcgen05.mma
// kind::tf32 with the 3xTF32 split of k_cgemm_tc.cu (fp32-level accuracy).
//
// Persistent CTAs (one per SM), warp-specialised like the contraction:
//   warp 0      producer (lane r: row r): one cp.async.bulk per input row
//               segment of the tile (kx*ky rows of 128 + kz - 1 floats; the
//               16-byte-aligned superset, its offset recorded per slot) into
//               an 8-slot ring, completion by mbarrier transaction bytes;
//   warps 8-11  converters: row m gathers its k^3 taps from the staged rows,
//               splits them into tf32 hi/lo and writes them to TMEM (A of
//               buffer t % 2);
//   warp 1      MMA issuer: 3 * K/8 MMAs into accumulator buffer t % 2;
//   warps 4-7,  epilogue, one warpgroup per accumulator buffer: tcgen05.ld,
//   12-15       bias + ReLU, stores -- lane m writes
//               voxel z0 + m of each map, so every store instruction writes a
//               whole 128-byte row segment (unlike the contraction's pieces).
// The pre-split W (N x K, hi/lo, UMMA K-major layout) and the bias stay in
// shared memory for the CTA's lifetime; TMEM holds 2 accumulators of N
// columns and 2 A buffers of 2K columns (<= 416 of 512).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "async.cuh"
#include "common.cuh"
#include "tcgen05.cuh"

namespace vxg {
namespace {

using namespace tc;

constexpr int DT_THREADS = 512;  // 16 warps: two epilogue warpgroups
constexpr int DT_NS = 8;     // staging slots
constexpr int DT_RS = 140;   // staged row stride (floats): the 16-byte superset of
                             // 128 + kz - 1 floats (up to 3 more) fits for kz <= 10
constexpr int DT_ROWS = 16;  // kx * ky <= 16

struct DtGeom {
  const float* in;
  const float* w;  // [N][kvol] (f = 1)
  const float* bias;
  float* out;      // [S][N][ox][oy][opz]
  int64_t S;
  int nx, ny, nz, ipz;
  int kx, ky, kz, kvol;
  int ox, oy, oz, opz;
  int ztiles;
  int64_t tiles;
  int relu;
  long long* prof;  // VXG_DT_PROF: per-CTA role cycle counters
};

template <int N, int K>
struct DtCfg {
  static constexpr int B_MAT = N * TC_KC * 4;
  static constexpr int W_BYTES = (K / TC_KC) * 2 * B_MAT;
  static constexpr int SLOT = DT_ROWS * DT_RS * 4;
  static constexpr int OFF_BIAS = 512;   // N floats
  static constexpr int OFF_TAPS = 1024;  // K ints: staged-row offset of tap q (-1: padding)
  static constexpr int OFF_TROW = 1280;  // K ints: staged row of tap q
  static constexpr int OFF_SHIFT = 1536; // [slot][row] ints: where a staged row's z0 lands (16-byte path)
  static constexpr int OFF_W = 2048;  // (shift table: DT_NS x 16 ints = 512 B)
  static constexpr int OFF_RING = OFF_W + W_BYTES;
  static constexpr int SMEM = OFF_RING + DT_NS * SLOT;
  // more than half an SM's shared memory: one CTA per SM, so the 512-column
  // TMEM allocation never waits on a co-resident CTA
  static constexpr int SMEM_LAUNCH = SMEM > 120 * 1024 ? SMEM : 120 * 1024;
  static constexpr int ACC = 0;           // accumulators: columns [b N, b N + N)
  static constexpr int ABUF = 2 * N;      // A buffer b: hi [ABUF + 2K b, + K), lo [+ K, + 2K)
  static_assert(2 * N + 4 * K <= 512, "TMEM columns");
};

template <int NV>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&u)[NV]);

template <>
__device__ __forceinline__ void tmem_st<8>(uint32_t t, const uint32_t (&u)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(t), "r"(u[0]),
               "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]));
}

template <>
__device__ __forceinline__ void tmem_st<32>(uint32_t t, const uint32_t (&u)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {"
      "%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(t),
      "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]), "r"(u[8]),
      "r"(u[9]), "r"(u[10]), "r"(u[11]), "r"(u[12]), "r"(u[13]), "r"(u[14]), "r"(u[15]), "r"(u[16]),
      "r"(u[17]), "r"(u[18]), "r"(u[19]), "r"(u[20]), "r"(u[21]), "r"(u[22]), "r"(u[23]), "r"(u[24]),
      "r"(u[25]), "r"(u[26]), "r"(u[27]), "r"(u[28]), "r"(u[29]), "r"(u[30]), "r"(u[31]));
}

template <int N, int K>
__global__ void __launch_bounds__(DT_THREADS, 1) direct_tc_kernel(DtGeom g) {
  using C = DtCfg<N, K>;
  constexpr int KC = K < 32 ? K : 32;  // converter chunk (TMEM store width)
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* slot_empty = full + DT_NS;
  uint64_t* ready = slot_empty + DT_NS;  // [2]
  uint64_t* a_empty = ready + 2;         // [2]
  uint64_t* acc_full = a_empty + 2;      // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* sbias = reinterpret_cast<float*>(smem + C::OFF_BIAS);
  int* staps = reinterpret_cast<int*>(smem + C::OFF_TAPS);
  int* sshift = reinterpret_cast<int*>(smem + C::OFF_SHIFT);
  int* strow = reinterpret_cast<int*>(smem + C::OFF_TROW);
  uint8_t* sw = smem + C::OFF_W;
  float* ring = reinterpret_cast<float*>(smem + C::OFF_RING);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t my_tiles = (g.tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;

  // W (N x K, zero taps past kvol) -> tf32 hi/lo matrices per K step; bias
  for (int e = tid; e < N * K; e += DT_THREADS) {
    const int j = e / K, q = e % K;
    const float v = q < g.kvol ? __ldg(g.w + int64_t(j) * g.kvol + q) : 0.f;
    float h, l;
    split_tf32(v, h, l);
    const int ks = q / TC_KC, kk = q % TC_KC;
    const int off = tile_off(j, kk >> 2) + (kk & 3) * 4;
    *reinterpret_cast<float*>(sw + (ks * 2 + 0) * C::B_MAT + off) = h;
    *reinterpret_cast<float*>(sw + (ks * 2 + 1) * C::B_MAT + off) = l;
  }
  for (int j = tid; j < N; j += DT_THREADS) sbias[j] = __ldg(g.bias + j);
  // in[p + k-1-q] (true convolution): tap q = (qx, qy, qz) reads staged row
  // (kx-1-qx, ky-1-qy) at column m + kz-1-qz
  for (int q = tid; q < K; q += DT_THREADS) {
    int off = -1, row = 0;
    if (q < g.kvol) {
      const int qz = q % g.kz, qy = (q / g.kz) % g.ky, qx = q / (g.kz * g.ky);
      row = (g.kx - 1 - qx) * g.ky + (g.ky - 1 - qy);
      off = row * DT_RS + (g.kz - 1 - qz);
    }
    staps[q] = off;
    strow[q] = row;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 32) {
    for (int s = 0; s < DT_NS; ++s) {
      mbar_init(&full[s], 1);  // the producer's arrive.expect_tx (+ the copies' transaction bytes)
      mbar_init(&slot_empty[s], 128);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ready[b], 128);
      mbar_init(&a_empty[b], 1);
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  // W was written through the generic proxy; the MMAs read it through the async one
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_slot;

  const bool small = g.tiles < (int64_t(1) << 31);
  auto decode = [&](int64_t lt, int64_t& s, int& x, int& y, int& z0) {
    if (small) {  // 32-bit division (the 64-bit one is a long software sequence)
      int t = int(blockIdx.x + lt * gridDim.x);
      z0 = (t % g.ztiles) * TC_M;
      t /= g.ztiles;
      y = t % g.oy;
      t /= g.oy;
      x = t % g.ox;
      s = t / g.ox;
      return;
    }
    int64_t t = blockIdx.x + lt * gridDim.x;
    z0 = int(t % g.ztiles) * TC_M;
    t /= g.ztiles;
    y = int(t % g.oy);
    t /= g.oy;
    x = int(t % g.ox);
    s = t / g.ox;
  };
  const int nrows = g.kx * g.ky, rlen = TC_M + g.kz - 1;

  if (warp == 0) {
    // ---------------- producer: one thread, one bulk copy per staged row ----------------
    // The copy engine moves the 16-byte-aligned superset of each row segment
    // ([o - sh, ...), sh = o mod 4) and signals the slot's mbarrier by
    // transaction bytes; the converters read the row at +sh.  Floats past nz
    // inside the last 16 bytes feed only outputs past oz, which are never
    // stored.
    long long pwt = 0;
    const long long pstart = clock64();
    // lane r < kx*ky owns staged row r: the row requests of a tile are issued
    // by different threads in parallel (one thread issuing all 16 in turn
    // was the kernel's bound)
    const int r = lane;
    const int aa = r < nrows ? r / g.ky : 0, bb = r < nrows ? r % g.ky : 0;
    const int64_t roff = (int64_t(aa) * g.ny + bb) * g.ipz;
    for (int64_t lt = 0; lt < my_tiles; ++lt) {
      const int s = int(lt % DT_NS);
      const long long pw0 = clock64();
      if (lt >= DT_NS) mbar_wait(&slot_empty[s], uint32_t((lt / DT_NS - 1) & 1));
      pwt += clock64() - pw0;
      int64_t si;
      int x, y, z0;
      decode(lt, si, x, y, z0);
      float* dst = ring + s * (DT_ROWS * DT_RS);
      const int64_t o = ((si * g.nx + x) * int64_t(g.ny) + y) * g.ipz + z0 + roff;
      const int sh = int(o & 3);
      const int64_t oa = o - sh;
      const int64_t need = std::min<int64_t>(int64_t(rlen), int64_t(g.nz - z0)) + sh;  // floats from oa
      const uint32_t nb = r < nrows ? uint32_t(((need + 3) >> 2) << 4) : 0u;
      if (r < nrows) sshift[s * DT_ROWS + r] = sh;
      // total bytes of the tile's rows (lanes >= nrows contribute 0)
      uint32_t bytes = nb;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, d);
      __syncwarp();  // orders the shift entries before lane 0's releasing arrive
      if (lane == 0) mbar_arrive_expect_tx(&full[s], bytes);
      __syncwarp();
      if (r < nrows) bulk_copy(dst + r * DT_RS, g.in + oa, nb, &full[s]);
    }
    if (g.prof && lane == 0) {
      g.prof[blockIdx.x * 8 + 0] = pwt;
      g.prof[blockIdx.x * 8 + 1] = clock64() - pstart;
    }
  } else if (warp >= 8 && warp < 12) {
    // ---------------- converters: thread m owns output voxel z0 + m ----------------
    const int m = tid - 256;
    const uint32_t lane_base = tmem + (uint32_t((warp & 3) * 32) << 16);
    long long cwf = 0, cwa = 0;
    for (int64_t lt = 0; lt < my_tiles; ++lt) {
      const int s = int(lt % DT_NS), b = int(lt & 1);
      const long long c0 = clock64();
      mbar_wait(&full[s], uint32_t((lt / DT_NS) & 1));
      const long long c1 = clock64();
      if (lt >= 2) mbar_wait(&a_empty[b], uint32_t((lt / 2 - 1) & 1));
      cwf += c1 - c0;
      cwa += clock64() - c1;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const float* src = ring + s * (DT_ROWS * DT_RS) + m;
      const int* shs = sshift + s * DT_ROWS;
#pragma unroll 1
      for (int q0 = 0; q0 < K; q0 += KC) {
        uint32_t hi[KC], lo[KC];
#pragma unroll
        for (int i = 0; i < KC; ++i) {
          const int off = staps[q0 + i];
          const float v = off >= 0 ? src[off + shs[strow[q0 + i]]] : 0.f;
          float h, l;
          split_tf32(v, h, l);
          hi[i] = __float_as_uint(h);
          lo[i] = __float_as_uint(l);
        }
        const uint32_t col = uint32_t(C::ABUF + 2 * K * b + q0);
        tmem_st<KC>(lane_base + col, hi);
        tmem_st<KC>(lane_base + col + K, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::);
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(&slot_empty[s]);
      mbar_arrive(&ready[b]);
    }
    if (g.prof && m == 0) {
      g.prof[blockIdx.x * 8 + 2] = cwf;
      g.prof[blockIdx.x * 8 + 3] = cwa;
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32<N>(false);
      const uint32_t wbase = smem_u32(sw);
      long long mwr = 0, mwe = 0;
      for (int64_t lt = 0; lt < my_tiles; ++lt) {
        const int b = int(lt & 1);
        const long long c0 = clock64();
        mbar_wait(&ready[b], uint32_t((lt / 2) & 1));
        const long long c1 = clock64();
        if (lt >= 2) mbar_wait(&acc_empty[b], uint32_t((lt / 2 - 1) & 1));
        mwr += c1 - c0;
        mwe += clock64() - c1;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const uint32_t d = tmem + uint32_t(C::ACC + N * b);
        const uint32_t ahi = tmem + uint32_t(C::ABUF + 2 * K * b);
#pragma unroll
        for (int ks = 0; ks < K / TC_KC; ++ks) {
          const uint64_t bhi = umma_desc(wbase + (ks * 2 + 0) * C::B_MAT);
          const uint64_t blo = umma_desc(wbase + (ks * 2 + 1) * C::B_MAT);
          const uint32_t a_h = ahi + uint32_t(ks * TC_KC), a_l = a_h + uint32_t(K);
          mma_tf32_ta(d, a_h, bhi, idesc, ks > 0 ? 1u : 0u);
          mma_tf32_ta(d, a_h, blo, idesc, 1u);
          mma_tf32_ta(d, a_l, bhi, idesc, 1u);
        }
        umma_commit(&a_empty[b]);
        umma_commit(&acc_full[b]);
      }
      if (g.prof) {
        g.prof[blockIdx.x * 8 + 4] = mwr;
        g.prof[blockIdx.x * 8 + 5] = mwe;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: warps 4-7 drain accumulator 0 (even tiles),
    // warps 12-15 accumulator 1 (odd tiles) ----------------
    const int eg = warp >= 12 ? 1 : 0;
    const int m = (warp & 3) * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t((warp & 3) * 32) << 16);
    const int64_t chan = int64_t(g.ox) * g.oy * g.opz;
    long long ewt = 0;
    for (int64_t lt = eg; lt < my_tiles; lt += 2) {
      const int b = eg;
      int64_t si;
      int x, y, z0;
      decode(lt, si, x, y, z0);
      const long long e0 = clock64();
      mbar_wait(&acc_full[b], uint32_t((lt / 2) & 1));
      ewt += clock64() - e0;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const int gz = z0 + m;
      float* o = g.out + si * N * chan + (int64_t(x) * g.oy + y) * g.opz + gz;
#pragma unroll 1
      for (int j0 = 0; j0 < N; j0 += 16) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
            "[%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15])
            : "r"(lane_base + uint32_t(C::ACC + N * b + j0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
        if (gz < g.oz) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const float r = __uint_as_float(v[jj]) + sbias[j0 + jj];
            o[int64_t(j0 + jj) * chan] = g.relu ? (r > 0.f ? r : 0.f) : r;  // activate (layers.hpp:105-108)
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(&acc_empty[b]);
    }
    if (g.prof && m == 0 && eg == 0) {
      g.prof[blockIdx.x * 8 + 6] = ewt;
      g.prof[blockIdx.x * 8 + 7] = my_tiles;
    }
  }
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

template <int N, int K>
void run_dt(Ctx* c, const DtGeom& g) {
  using C = DtCfg<N, K>;
  static PerDeviceOnce configured;
  if (configured.first()) {
    VXG_CUDA_CHECK(cudaFuncSetAttribute(direct_tc_kernel<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        C::SMEM_LAUNCH));
  }
  const unsigned grid = unsigned(std::min<int64_t>(g.tiles, c->num_sms));
  static const bool prof = std::getenv("VXG_DT_PROF") != nullptr;
  DtGeom h = g;
  long long* dprof = nullptr;
  if (prof) {
    VXG_CUDA_CHECK(cudaMalloc(&dprof, size_t(grid) * 8 * sizeof(long long)));
    VXG_CUDA_CHECK(cudaMemset(dprof, 0, size_t(grid) * 8 * sizeof(long long)));
    h.prof = dprof;
  }
  direct_tc_kernel<N, K><<<grid, DT_THREADS, C::SMEM_LAUNCH, c->stream>>>(h);
  c->counted();
  check_launch("direct_tc_kernel");
  if (prof) {
    std::vector<long long> v(size_t(grid) * 8);
    VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    VXG_CUDA_CHECK(cudaMemcpy(v.data(), dprof, v.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(dprof);
    double a[8] = {0};
    for (unsigned bb = 0; bb < grid; ++bb)
      for (int k = 0; k < 8; ++k) a[k] += double(v[bb * 8 + k]) / grid;
    std::fprintf(stderr,
                 "[dtprof] N=%d tiles/CTA %.0f total %.3gM | producer wait-slot %.3gM | converter wait-data %.3gM "
                 "wait-A %.3gM | mma wait-ready %.3gM wait-acc %.3gM | epilogue wait %.3gM  (per tile: %.0f cyc)\n",
                 N, a[7], a[1] / 1e6, a[0] / 1e6, a[2] / 1e6, a[3] / 1e6, a[4] / 1e6, a[5] / 1e6, a[6] / 1e6,
                 a[1] / std::max(1.0, a[7]));
  }
}

template <int N>
void run_dt_k(Ctx* c, const DtGeom& g) {
  const int K = (g.kvol + 7) / 8 * 8;
  if (K <= 8)
    run_dt<N, 8>(c, g);
  else if (K <= 32)
    run_dt<N, 32>(c, g);
  else
    run_dt<N, 64>(c, g);
}

}  // namespace

bool direct_tc_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VXG_DIRECT_TC");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return on;
}

// The kernel is bound by its input staging (~3 us per 128-voxel tile at
// k = 4: 16 row requests, no reuse between neighbouring rows), whatever the
// channel block: it beats the FFMA kernel from 48 maps per launch on
// (80 maps: 6.6-7.1 vs 12.4 ms at 330^3), not below.
int64_t direct_tc_min_maps() {
  static const int64_t v = [] {
    const char* e = std::getenv("VXG_DIRECT_TC_MIN");
    return e ? int64_t(std::atoll(e)) : int64_t(48);
  }();
  return v;
}

bool direct_tc_supported(int64_t f, int64_t fo, V3 k, const void* in) {
  return direct_tc_enabled() && f == 1 && fo % 16 == 0 && fo >= direct_tc_min_maps() && fo <= 80 &&
         k.x * k.y <= DT_ROWS &&
         k.vol() <= 64 && TC_M + k.z - 1 + 3 <= DT_RS &&  // + 3: 16-byte superset of the row
         (reinterpret_cast<uintptr_t>(in) & 15) == 0;  // bulk copies of 16-byte-aligned row supersets
}

// f = 1 direct convolution on the tensor cores (callers check direct_tc_supported)
void launch_direct_tc(Ctx* c, const float* in, i64 S, V3 n, const float* w, i64 fo, V3 k, const float* bias,
                      bool relu, float* out, i64 ipz, i64 opz) {
  DtGeom g{};
  g.in = in; g.w = w; g.bias = bias; g.out = out;
  g.S = S;
  g.nx = int(n.x); g.ny = int(n.y); g.nz = int(n.z);
  g.ipz = int(ipz > 0 ? ipz : n.z);
  g.kx = int(k.x); g.ky = int(k.y); g.kz = int(k.z);
  g.kvol = int(k.vol());
  g.ox = int(n.x - k.x + 1); g.oy = int(n.y - k.y + 1); g.oz = int(n.z - k.z + 1);
  g.opz = int(opz > 0 ? opz : g.oz);
  g.ztiles = (g.oz + TC_M - 1) / TC_M;
  g.tiles = S * g.ox * g.oy * int64_t(g.ztiles);
  g.relu = relu ? 1 : 0;
  g.prof = nullptr;
  if (g.tiles == 0) return;
  const double vox = double(g.ox) * g.oy * g.oz;
  KScope ks(c, VXG_K_DIRECT, 2.0 * double(S) * fo * vox * double(g.kvol),
            4.0 * (double(S) * g.nx * g.ny * g.nz + double(S) * fo * vox + double(fo) * g.kvol));
  switch (fo) {
    case 16: run_dt_k<16>(c, g); break;
    case 32: run_dt_k<32>(c, g); break;
    case 48: run_dt_k<48>(c, g); break;
    case 64: run_dt_k<64>(c, g); break;
    case 80: run_dt_k<80>(c, g); break;
    default: throw invalid("direct_tc: unsupported map count");
  }
}

}  // namespace vxg
