// K3 on the 5th-generation tensor cores: the per-frequency complex
// contraction Y[w](m, i) = sum_j X[w](m, j) W[w](i, j) (the MAC of
// proj/include/voxin/layers.hpp:245-251, 330-344) as tcgen05.mma kind::tf32
// with a 3xTF32 split (a*b ~ a_hi*b_hi + a_hi*b_lo + a_lo*b_hi, fp32
// accumulation in TMEM), which keeps fp32-level accuracy (~2^-21 relative per
// product) inside the 1e-4 parity tolerance.
//
// Complex -> real: for each frequency w, with X = Xr + i Xi and W = Wr + i Wi,
//   Dr += Xr Wr^T - Xi Wi^T      (the minus via the instruction's B-negate bit)
//   Di += Xr Wi^T + Xi Wr^T
// M = 128 rows (tiles x batch), N = fo output maps, K = input maps in chunks
// of 8 (one tf32 MMA K-step).  Spectra use 128-byte lines of 16 frequencies
// ([w/16][row][channel][w%16]); a CTA tile is one frequency PAIR (a 16-byte
// piece of each line) x 128 rows, so 4 accumulators of N columns = 4*fo <= 512
// TMEM columns.  Tiles are ordered (line block, m-block, pair) with the pair
// fastest: the 8 CTAs reading pieces of the same lines run concurrently and
// share them through L2.
//
// Y is written line-major (16-byte pieces, like X) or, for the CTA-pair
// inverse transform, pair-major ([w/2][row][map][2]): then a warp-local
// transpose turns the epilogue's stores into whole-line writes.
//
// Persistent, warp-specialised pipeline over a flat stream of (tile, K-chunk)
// items and a 3-slot shared-memory ring (raw X chunk | pre-split W chunk |
// split X chunk per slot), handshakes on mbarriers:
//   warp 0        producer: cp.async of the raw X chunk (rows padded to
//                 144 B) + one bulk copy of the W chunk (already tf32 hi/lo in
//                 the UMMA layout, written once per layer by wsplit_kernel);
//                 completion tracked on full[slot];
//   warps 8-11    converters: split X into tf32 hi/lo and write it to
//                 tensor memory (row = TMEM lane, 64 columns per slot), so
//                 the MMAs take A from TMEM and read only W from shared
//                 memory (A and B from shared memory made the K = 8 MMAs
//                 shared-memory-bandwidth bound), arrive on ready[slot];
//   warp 1        MMA issuer (one thread): 24 tcgen05.mma per chunk, commit to
//                 empty[slot] (frees the slot) and, after a tile's last chunk,
//                 to tmem_full;
//   warps 4-7     epilogue (TMEM lane quadrants 0-3): tcgen05.ld, 16-byte
//                 stores of the Y pieces, arrive on tmem_empty.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "async.cuh"
#include "common.cuh"
#include "fftconv.hpp"
#include "tcgen05.cuh"

namespace vxg {
namespace {

using namespace tc;
constexpr int TC_SLOTS = 3;
constexpr int TC_THREADS = 384;  // 12 warps
constexpr int RAW_ROW = 144;     // padded raw-row stride (bytes)

template <int FO>
struct TcCfg {
  static constexpr int A_MAT = TC_M * TC_KC * 4;   // one 128 x 8 tf32 matrix
  static constexpr int B_MAT = FO * TC_KC * 4;     // one FO x 8 tf32 matrix
  static constexpr int B_CHUNK = 8 * B_MAT;        // pre-split W chunk (w, re/im, hi/lo)
  static constexpr int RAW_A = TC_M * RAW_ROW;
  static constexpr int OFF_W = RAW_A;
  static constexpr int SLOT = RAW_A + B_CHUNK;     // (split X lives in TMEM)
  static constexpr int ACOL = 4 * FO;              // TMEM column of A slot 0 (64 columns per slot)
  static constexpr int STAGE = 4 * 4096;  // pair-major epilogue: 4 KB transpose tile per warp
  static constexpr int SMEM = TC_SLOTS * SLOT + STAGE + 128;
};

// ---- one-time W preparation: raw [w/16][i][j][16] complex -> per (pair, chunk)
// the 8 matrices (w, re/im, hi/lo) of FO x 8 tf32 in the UMMA layout.
template <int FO>
__global__ void wsplit_kernel(const float4* __restrict__ raw, uint8_t* __restrict__ out,
                              int64_t npairs, int f) {
  using C = TcCfg<FO>;
  const int nchunks = f / TC_KC;
  const int64_t total = npairs * nchunks * FO * 2;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int hk = int(t & 1);
    const int i = int((t >> 1) % FO);
    const int64_t pc = (t >> 1) / FO;  // pair * nchunks + kc
    const int kc = int(pc % nchunks);
    const int64_t pair = pc / nchunks;
    const int64_t wb = pair >> 3;
    const int pip = int(pair & 7);
    const float4* src = raw + ((wb * FO + i) * f + kc * TC_KC + 4 * hk) * 8 + pip;
    float4 v[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) v[kk] = src[kk * 8];
    uint8_t* dst = out + pc * C::B_CHUNK;
#pragma unroll
    for (int wc = 0; wc < 4; ++wc) {
      float h[4], l[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const float x = wc == 0 ? v[kk].x : wc == 1 ? v[kk].y : wc == 2 ? v[kk].z : v[kk].w;
        split_tf32(x, h[kk], l[kk]);
      }
      *reinterpret_cast<float4*>(dst + (wc * 2 + 0) * C::B_MAT + tile_off(i, hk)) = make_float4(h[0], h[1], h[2], h[3]);
      *reinterpret_cast<float4*>(dst + (wc * 2 + 1) * C::B_MAT + tile_off(i, hk)) = make_float4(l[0], l[1], l[2], l[3]);
    }
  }
}

struct TileCoord {
  int64_t wb, m0, pair;
  int pip;
};

template <int FO>
__global__ void __launch_bounds__(TC_THREADS, 1) cgemm_tc_kernel(GemmArgs a) {
  using C = TcCfg<FO>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ystage = smem + TC_SLOTS * C::SLOT;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC_SLOTS * C::SLOT + C::STAGE);
  uint64_t* ready = full + TC_SLOTS;
  uint64_t* empty = ready + TC_SLOTS;
  uint64_t* tmem_full = empty + TC_SLOTS;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nchunks = a.f / TC_KC;
  const int64_t ntiles = int64_t(a.mblocks) * a.npairs;
  const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t nitems = my_tiles * nchunks;

  auto coord = [&](int64_t local_tile) {
    const int64_t tile = blockIdx.x + local_tile * gridDim.x;
    TileCoord tc;
    tc.pip = int(tile & 7);
    const int64_t rest = tile >> 3;
    tc.m0 = (rest % a.mblocks) * TC_M;
    tc.wb = rest / a.mblocks;
    tc.pair = tc.wb * 8 + tc.pip;
    return tc;
  };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 32) {
    for (int s = 0; s < TC_SLOTS; ++s) {
      mbar_init(&full[s], 32 + 1);  // 32 producer lanes (cp.async) + the W bulk copy arrive
      mbar_init(&ready[s], 128);    // converter threads
      mbar_init(&empty[s], 1);      // MMA commit
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 128);     // epilogue threads
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- producer ----------------
    const float4* xsrc = reinterpret_cast<const float4*>(a.X);  // one float4 = 2 complex
    long long pw = 0;
    for (int64_t g = 0; g < nitems; ++g) {
      const int s = int(g % TC_SLOTS);
      const long long t0 = a.prof ? clock64() : 0;
      if (g >= TC_SLOTS) mbar_wait(&empty[s], uint32_t((g / TC_SLOTS - 1) & 1));
      if (a.prof) pw += clock64() - t0;
      const TileCoord tc = coord(g / nchunks);
      const int kc = int(g % nchunks);
      uint8_t* slot = smem + s * C::SLOT;
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[s], C::B_CHUNK);
        bulk_copy(slot + C::OFF_W,
                  reinterpret_cast<const uint8_t*>(a.W) + (tc.pair * nchunks + kc) * int64_t(C::B_CHUNK),
                  C::B_CHUNK, &full[s]);
      }
#pragma unroll 4
      for (int u = lane; u < TC_M * TC_KC; u += 32) {
        const int row = u >> 3, jj = u & 7;
        const bool ok = tc.m0 + row < a.M;
        const float4* src =
            ok ? xsrc + ((tc.wb * a.mstride + tc.m0 + row) * a.f + kc * TC_KC + jj) * 8 + tc.pip : xsrc;
        cp_async16(slot + row * RAW_ROW + jj * 16, src, ok);
      }
      cp_async_arrive_noinc(&full[s]);
    }
    if (a.prof && lane == 0) a.prof[blockIdx.x * 8 + 0] = pw;
  } else if (warp >= 8) {
    // ---------------- converters: thread c owns row c ----------------
    const int c = tid - 256;
    long long cw = 0, cb = 0;
    for (int64_t g = 0; g < nitems; ++g) {
      const int s = int(g % TC_SLOTS);
      const long long t0 = a.prof ? clock64() : 0;
      mbar_wait(&full[s], uint32_t((g / TC_SLOTS) & 1));
      const long long t1 = a.prof ? clock64() : 0;
      cw += t1 - t0;
      uint8_t* slot = smem + s * C::SLOT;
      const uint8_t* raw = slot + c * RAW_ROW;
      // split X row c into tf32 hi/lo and write it to TMEM lane c: matrix
      // (w, re/im, hi/lo) = columns ACOL + 64 s + 8 * ((w*2 + comp)*2 + h) + channel
      uint32_t u[64];
#pragma unroll
      for (int hk = 0; hk < 2; ++hk) {
        float4 v[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) v[kk] = *reinterpret_cast<const float4*>(raw + (4 * hk + kk) * 16);
#pragma unroll
        for (int wc = 0; wc < 4; ++wc) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const float x = wc == 0 ? v[kk].x : wc == 1 ? v[kk].y : wc == 2 ? v[kk].z : v[kk].w;
            float h, l;
            split_tf32(x, h, l);
            u[(wc * 2 + 0) * 8 + 4 * hk + kk] = __float_as_uint(h);
            u[(wc * 2 + 1) * 8 + 4 * hk + kk] = __float_as_uint(l);
          }
        }
      }
      const uint32_t ta = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(C::ACOL + 64 * s);
      if (!(a.dbg & 1)) asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {"
          "%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,"
          "%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,"
          "%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};\n" ::"r"(ta),
          "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]),
          "r"(u[8]), "r"(u[9]), "r"(u[10]), "r"(u[11]), "r"(u[12]), "r"(u[13]), "r"(u[14]), "r"(u[15]),
          "r"(u[16]), "r"(u[17]), "r"(u[18]), "r"(u[19]), "r"(u[20]), "r"(u[21]), "r"(u[22]), "r"(u[23]),
          "r"(u[24]), "r"(u[25]), "r"(u[26]), "r"(u[27]), "r"(u[28]), "r"(u[29]), "r"(u[30]), "r"(u[31]),
          "r"(u[32]), "r"(u[33]), "r"(u[34]), "r"(u[35]), "r"(u[36]), "r"(u[37]), "r"(u[38]), "r"(u[39]),
          "r"(u[40]), "r"(u[41]), "r"(u[42]), "r"(u[43]), "r"(u[44]), "r"(u[45]), "r"(u[46]), "r"(u[47]),
          "r"(u[48]), "r"(u[49]), "r"(u[50]), "r"(u[51]), "r"(u[52]), "r"(u[53]), "r"(u[54]), "r"(u[55]),
          "r"(u[56]), "r"(u[57]), "r"(u[58]), "r"(u[59]), "r"(u[60]), "r"(u[61]), "r"(u[62]), "r"(u[63]));
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::);
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(&ready[s]);
      if (a.prof) cb += clock64() - t1;
    }
    if (a.prof && c == 0) {
      a.prof[blockIdx.x * 8 + 1] = cw;
      a.prof[blockIdx.x * 8 + 2] = cb;
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      long long me = 0, mr = 0;
      const long long tstart = a.prof ? clock64() : 0;
      for (int64_t g = 0; g < nitems; ++g) {
        const int s = int(g % TC_SLOTS);
        const int kc = int(g % nchunks);
        const int64_t t = g / nchunks;
        const long long t0 = a.prof ? clock64() : 0;
        if (kc == 0 && t > 0) mbar_wait(tmem_empty, uint32_t((t - 1) & 1));  // epilogue drained TMEM
        const long long t1 = a.prof ? clock64() : 0;
        mbar_wait(&ready[s], uint32_t((g / TC_SLOTS) & 1));
        if (a.prof) {
          me += t1 - t0;
          mr += clock64() - t1;
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const uint32_t slot = smem_u32(smem + s * C::SLOT);
        const uint32_t sb = slot + C::OFF_W;
        const uint32_t ta = tmem + uint32_t(C::ACOL + 64 * s);
        const uint32_t first = kc > 0 ? 1u : 0u;
        // the four accumulators (w0 re, w0 im, w1 re, w1 im) round-robin, so
        // consecutive MMAs never target the same accumulator
        auto am = [&](int w, int cc, int h) { return ta + uint32_t(((w * 2 + cc) * 2 + h) * 8); };
        auto bm = [&](int w, int cc, int h) { return umma_desc(sb + ((w * 2 + cc) * 2 + h) * C::B_MAT); };
        const uint32_t ip = idesc_tf32<FO>(false), in = idesc_tf32<FO>(true);
        // term list per accumulator: (A comp, A half, B comp, B half, negate)
        constexpr int TR[6][5] = {{0, 0, 0, 0, 0}, {0, 0, 0, 1, 0}, {0, 1, 0, 0, 0},
                                  {1, 0, 1, 0, 1}, {1, 0, 1, 1, 1}, {1, 1, 1, 0, 1}};  // Dr = XrWr - XiWi
        constexpr int TI[6][5] = {{0, 0, 1, 0, 0}, {0, 0, 1, 1, 0}, {0, 1, 1, 0, 0},
                                  {1, 0, 0, 0, 0}, {1, 0, 0, 1, 0}, {1, 1, 0, 0, 0}};  // Di = XrWi + XiWr
#pragma unroll
        for (int k = 0; k < ((a.dbg & 4) ? 0 : 6); ++k) {
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const uint32_t dr = tmem + w * 2 * FO, di = dr + FO;
            const uint32_t acc = k == 0 ? first : 1u;
            mma_tf32_ta(dr, am(w, TR[k][0], TR[k][1]), bm(w, TR[k][2], TR[k][3]), TR[k][4] ? in : ip, acc);
            mma_tf32_ta(di, am(w, TI[k][0], TI[k][1]), bm(w, TI[k][2], TI[k][3]), TI[k][4] ? in : ip, acc);
          }
        }
        umma_commit(&empty[s]);                       // slot reusable once these MMAs finish
        if (kc == nchunks - 1) umma_commit(tmem_full);  // tile accumulated
      }
      if (a.prof) {
        a.prof[blockIdx.x * 8 + 3] = me;
        a.prof[blockIdx.x * 8 + 4] = mr;
        a.prof[blockIdx.x * 8 + 7] = clock64() - tstart;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: warp 4+q owns TMEM lanes 32q .. 32q+31 ----------------
    const int q = warp - 4;
    const int row = q * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t(q * 32) << 16);
    long long ew = 0, eb = 0;
    for (int64_t t = 0; t < my_tiles; ++t) {
      const long long t0 = a.prof ? clock64() : 0;
      mbar_wait(tmem_full, uint32_t(t & 1));
      const long long t1 = a.prof ? clock64() : 0;
      ew += t1 - t0;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const TileCoord tc = coord(t);
      const int64_t m = tc.m0 + row;
      if (a.ypair) {
        // pair-major Y ([pair][row][map] 16-byte pieces): a row's maps are
        // contiguous, so a warp-local transpose through shared memory (16-byte
        // chunks XOR-swizzled by row) lets every store instruction write four
        // whole 128-byte lines instead of 32 scattered pieces
        uint8_t* stg = ystage + q * 4096;
        float4* ybase = reinterpret_cast<float4*>(a.Y) + (tc.pair * a.mstride + tc.m0) * a.fo;
#pragma unroll 1
        for (int i0 = 0; i0 < FO; i0 += 8) {
          uint32_t v[4][8];
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const uint32_t col = (qq >> 1) * 2 * FO + (qq & 1) * FO + i0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                : "=r"(v[qq][0]), "=r"(v[qq][1]), "=r"(v[qq][2]), "=r"(v[qq][3]), "=r"(v[qq][4]),
                  "=r"(v[qq][5]), "=r"(v[qq][6]), "=r"(v[qq][7])
                : "r"(lane_base + col));
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
#pragma unroll
          for (int cc = 0; cc < 8; ++cc)
            *reinterpret_cast<float4*>(stg + lane * 128 + ((cc ^ (lane & 7)) << 4)) =
                make_float4(__uint_as_float(v[0][cc]), __uint_as_float(v[1][cc]), __uint_as_float(v[2][cc]),
                            __uint_as_float(v[3][cc]));
          __syncwarp();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int r = 4 * k + (lane >> 3), cc = lane & 7;
            const float4 piece = *reinterpret_cast<const float4*>(stg + r * 128 + ((cc ^ (r & 7)) << 4));
            if (tc.m0 + q * 32 + r < a.M && !(a.dbg & 2)) ybase[int64_t(q * 32 + r) * a.fo + i0 + cc] = piece;
          }
          __syncwarp();
        }
      } else {
      float4* yrow = reinterpret_cast<float4*>(a.Y) + (tc.wb * a.mstride + m) * a.fo * 8 + tc.pip;
#pragma unroll 1
      for (int i0 = 0; i0 < FO; i0 += 16) {
        uint32_t v[4][16];  // (w0 re, w0 im, w1 re, w1 im) x 16 maps
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const uint32_t col = (qq >> 1) * 2 * FO + (qq & 1) * FO + i0;
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
              "[%16];\n"
              : "=r"(v[qq][0]), "=r"(v[qq][1]), "=r"(v[qq][2]), "=r"(v[qq][3]), "=r"(v[qq][4]),
                "=r"(v[qq][5]), "=r"(v[qq][6]), "=r"(v[qq][7]), "=r"(v[qq][8]), "=r"(v[qq][9]),
                "=r"(v[qq][10]), "=r"(v[qq][11]), "=r"(v[qq][12]), "=r"(v[qq][13]), "=r"(v[qq][14]),
                "=r"(v[qq][15])
              : "r"(lane_base + col));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
        if (m < a.M && !(a.dbg & 2)) {
#pragma unroll
          for (int ii = 0; ii < 16; ++ii)
            yrow[(i0 + ii) * 8] = make_float4(__uint_as_float(v[0][ii]), __uint_as_float(v[1][ii]),
                                              __uint_as_float(v[2][ii]), __uint_as_float(v[3][ii]));
        }
      }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(tmem_empty);
      if (a.prof) eb += clock64() - t1;
    }
    if (a.prof && q == 0 && lane == 0) {
      a.prof[blockIdx.x * 8 + 5] = ew;
      a.prof[blockIdx.x * 8 + 6] = eb;
    }
  }
  // warps 2-3 have no role
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

template <int FO>
void tc_t(Ctx* c, GemmArgs a) {
  using C = TcCfg<FO>;
  static PerDeviceOnce configured;
  if (configured.first()) {
    VXG_CUDA_CHECK(cudaFuncSetAttribute(cgemm_tc_kernel<FO>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  }
  a.mblocks = int((a.M + TC_M - 1) / TC_M);
  const int64_t ntiles = int64_t(a.mblocks) * a.npairs;  // npairs = 8 per 16-frequency line
  const unsigned grid = unsigned(std::min<int64_t>(ntiles, c->num_sms));
  // VXG_TC_PROF=1: per-role wait / busy cycles (clock64) printed per launch
  static const bool prof = std::getenv("VXG_TC_PROF") != nullptr;
  static const int dbg = std::getenv("VXG_TC_DBG") ? std::atoi(std::getenv("VXG_TC_DBG")) : 0;
  a.dbg = dbg;
  long long* dprof = nullptr;
  if (prof) {
    VXG_CUDA_CHECK(cudaMalloc(&dprof, size_t(grid) * 8 * sizeof(long long)));
    VXG_CUDA_CHECK(cudaMemset(dprof, 0, size_t(grid) * 8 * sizeof(long long)));
    a.prof = dprof;
  }
  cgemm_tc_kernel<FO><<<grid, TC_THREADS, C::SMEM, c->stream>>>(a);
  c->counted();
  check_launch("cgemm_tc_kernel");
  if (prof) {
    std::vector<long long> h(size_t(grid) * 8);
    VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    VXG_CUDA_CHECK(cudaMemcpy(h.data(), dprof, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(dprof);
    double m[8] = {0};
    for (unsigned b = 0; b < grid; ++b)
      for (int k = 0; k < 8; ++k) m[k] += double(h[b * 8 + k]) / grid;
    std::fprintf(stderr,
                 "[tcprof] M=%lld total %.3gM | producer wait %.3gM | converter wait %.3gM busy %.3gM | "
                 "mma wait-epilogue %.3gM wait-ready %.3gM | epilogue wait %.3gM busy %.3gM\n",
                 (long long)a.M, m[7] / 1e6, m[0] / 1e6, m[1] / 1e6, m[2] / 1e6, m[3] / 1e6, m[4] / 1e6,
                 m[5] / 1e6, m[6] / 1e6);
  }
}

template <int FO>
void wsplit_t(Ctx* c, const float2* raw, void* out, int64_t npairs, int f) {
  const int64_t total = npairs * (f / TC_KC) * FO * 2;
  wsplit_kernel<FO><<<grid_for(total, 256, int64_t(c->num_sms) * 16), 256, 0, c->stream>>>(
      reinterpret_cast<const float4*>(raw), static_cast<uint8_t*>(out), npairs, f);
  c->counted();
  check_launch("wsplit_kernel");
}

}  // namespace

// fo <= 80 keeps the 3-slot ring (raw X | split W | split X) inside 227 KB of smem
bool cgemm_tc_supported(int64_t f, int64_t fo) {
  return f % TC_KC == 0 && f >= TC_KC && fo % 16 == 0 && fo >= 16 && fo <= 80;
}

int64_t tc_wsplit_bytes(int64_t npairs, int64_t f, int64_t fo, bool quad) {
  if (quad) return q_wsplit_bytes(npairs, f, fo);
  return npairs * (f / TC_KC) * 8 * fo * TC_KC * 4;
}

#define VXG_TC_SWITCH(CALL)                                           \
  switch (fo) {                                                       \
    case 16: CALL(16); break;                                         \
    case 32: CALL(32); break;                                         \
    case 48: CALL(48); break;                                         \
    case 64: CALL(64); break;                                         \
    case 80: CALL(80); break;                                         \
    default: throw invalid("cgemm_tc: unsupported output map count"); \
  }

void tc_wsplit(Ctx* c, const float2* raw, void* out, int64_t npairs, int64_t f, int64_t fo, bool quad) {
  if (quad) return q_wsplit(c, raw, out, npairs, f, fo);
  KScope ks(c, VXG_K_KSPEC, 0.0, double(npairs) * f * fo * (16.0 + 32.0));
#define VXG_WS(F) wsplit_t<F>(c, raw, out, npairs, int(f))
  VXG_TC_SWITCH(VXG_WS)
#undef VXG_WS
}

// Y[w/16][row][fo][16] = X[w/16][row][f][16] . W (pre-split by tc_wsplit)
void launch_cgemm_tc(Ctx* c, const GemmArgs& a, int64_t npairs) {
  if (a.quad && !a.ypair) return launch_cgemm_q(c, a, npairs);
  const double nw = double(a.T) * a.T * (a.T / 2 + 1);
  KScope ks(c, VXG_K_CGEMM, 8.0 * double(a.M) * a.f * a.fo * nw,
            8.0 * nw * (double(a.M) * a.f + double(a.M) * a.fo + double(a.f) * a.fo));
  GemmArgs b = a;
  b.npairs = npairs;
  const int64_t fo = a.fo;
#define VXG_TC(F) tc_t<F>(c, b)
  VXG_TC_SWITCH(VXG_TC)
#undef VXG_TC
}

}  // namespace vxg
