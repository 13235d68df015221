// K3 on the 5th-generation tensor cores, quad-frequency tiles: the
// per-frequency complex contraction Y[w](m, i) = sum_j X[w](m, j) W[w](i, j)
// (the MAC of proj/include/voxin/layers.hpp:245-251, 330-344) on tcgen05.mma
// with fp32 accumulation in TMEM.  Each real product costs two MMAs: a
// kind::tf32 MMA for a_hi*b_hi and one kind::f16 MMA (K = 16) for both
// correction terms, [bf16(a_hi) | bf16(a_lo)] . [bf16(b_lo) ; bf16(b_hi)]
// (a_hi = a with 13 mantissa bits cleared, a_lo = a - a_hi).  The correction
// terms are ~2^-11 of the product, so their bf16 rounding adds ~2^-19 relative
// error per product; VXG_Q_3TF32=1 selects the 3xTF32 split instead
// (a_hi*b_hi + a_hi*b_lo + a_lo*b_hi, three tf32 MMAs).
//
// Why quads: spectra are line-major ([w/16][row][map][16 w], 128-byte lines,
// the layout the tile transforms read and write whole).  A store that fills a
// whole 32-byte sector runs at ~5 TB/s, a 16-byte half-sector store at ~1 TB/s
// (tools/micro/ystore.cu).  So a CTA tile owns 4 consecutive frequencies (one
// 32-byte sector of every line it writes) x 128 rows x half of the output maps
// (NS = fo / 2), and each MMA is the real-block product
//   [Dr | Di] += Xr [Wr | Wi] + Xi [-Wi | Wr]        (N = 2 NS = fo columns)
// with W stored once per part (hi; correction) as three N-blocks (-Wi, Wr, Wi):
// the B operand [-Wi | Wr] starts at block 0 and [Wr | Wi] at block 1.
//
// TMEM: four accumulators (one per frequency, fo columns each, <= 320) + three
// 64-column A slots.  The K loop of a tile runs in two passes (frequencies 0-1
// of the quad, then 2-3), each with its own accumulator pair, so the epilogue
// drains pass 0 (parking it in shared memory) while pass 1 multiplies, and
// stores the whole 32-byte sectors while the next tile's pass 0 multiplies.
//
// Persistent, warp-specialised pipeline over items (tile, pass, K chunk of 8
// input maps), handshakes on mbarriers:
//   warp 0 lane 0  X producer: per item one TMA box per channel line (the
//                  pass's 16-byte piece of 128 rows), staged [channel][row]
//                  so a converter thread per row reads conflict-free, into a
//                  ring of 6 items (fo = 80), freed by the converters as soon
//                  as they hold the item in registers;
//   warp 2 lane 0  W producer: one bulk copy of the item's pre-split W
//                  (written once per layer by q_wsplit_kernel) into a 3-deep
//                  ring shared with the TMEM A slots;
//   warps 8-15     converters, two groups taking alternate items (a thread
//                  per row each): split X into tf32 hi/lo, tcgen05.st into the
//                  item's TMEM A slot (row = lane), arrive on ready[slot];
//   warp 1         MMA issuer (one thread): 8 tcgen05.mma per item (12 with
//                  the 3xTF32 split), one
//                  commit per item (frees the A and W slot) and, after a pass's
//                  last chunk, acc_full[pass];
//   warps 4-7      epilogue (TMEM lane quadrants 0-3).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "fftconv.hpp"
#include "tcgen05.cuh"

namespace vxg {

void encode_tensor_map_f32(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
                           const uint64_t* strides, const uint32_t* box);

// VXG_Q_3TF32=1: the full 3xTF32 split (3 MMAs per product) instead of the
// tf32 + bf16-correction pair (the W layout follows the same switch)
bool q_bf16_correction() {
  const char* e = std::getenv("VXG_Q_3TF32");
  return !(e && std::strcmp(e, "0") != 0);
}

namespace {

using namespace tc;
constexpr int Q_THREADS = 512;  // 16 warps
// staged X box: [channel][row][16 B] (one TMA box per channel line), so a
// converter thread per row reads conflict-free; row-major staging needed a 9th
// padding line per row (1/9 more L2 reads, 7-9 % slower, profiles/r2_experiments.md §14)
constexpr int Q_RAW = TC_KC * TC_M * 16;

template <int FO>
struct QCfg {
  static constexpr int AS = 4 * FO + 4 * 64 <= 512 ? 4 : 3;  // A (TMEM) / W (smem) ring depth
  static constexpr int NS = FO / 2;                 // output maps per tile
  static constexpr int BMAT = 3 * NS * TC_KC * 4;   // (-Wi, Wr, Wi) x 8 channels, one hi/lo part
  static constexpr int WITEM = 4 * BMAT;            // 2 frequencies x hi/lo
  static constexpr int PARK_ROW = NS * 16 + 16;     // pass-0 results per row (+16: conflict-free)
  static constexpr int BAR_BYTES = 384;
  // staged-X ring: as deep as fits beside the W ring and the park (<= 8)
  static constexpr int RS_FIT = (232448 - BAR_BYTES - TC_M * PARK_ROW - AS * WITEM) / Q_RAW;
  static constexpr int RS = RS_FIT > 8 ? 8 : RS_FIT;
  static constexpr int OFF_W = RS * Q_RAW;
  static constexpr int OFF_PARK = OFF_W + AS * WITEM;
  static constexpr int OFF_BAR = OFF_PARK + TC_M * PARK_ROW;
  static constexpr int SMEM = OFF_BAR + BAR_BYTES;
  static constexpr int ACOL = 4 * FO;               // TMEM column of A slot 0
  static_assert((2 * RS + 3 * AS + 4) * 8 + 4 <= BAR_BYTES, "cgemm_q: barrier area");
};

// ---- one-time W preparation: raw [w/16][i][j][16] complex -> per item
// (pair p, half h, chunk kc) the matrices (w, hi/lo) x blocks (-Wi, Wr, Wi) of
// NS x 8 tf32 in the UMMA K-major layout.
template <int FO, bool BFC>
__global__ void q_wsplit_kernel(const float2* __restrict__ raw, uint8_t* __restrict__ out, int64_t npairs,
                                int f) {
  using C = QCfg<FO>;
  const int nch = f / TC_KC;
  // one thread per (p, h, kc, w, n, k-group of 4)
  const int64_t total = npairs * 2 * nch * 2 * C::NS * 2;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int kg = int(t & 1);
    int64_t r = t >> 1;
    const int n = int(r % C::NS);
    r /= C::NS;
    const int w = int(r & 1);
    r >>= 1;
    const int kc = int(r % nch);
    r /= nch;
    const int h = int(r & 1);
    const int64_t p = r >> 1;
    const int64_t om = 2 * p + w;  // frequency
    const int i = h * C::NS + n;
    float re[4], im[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int j = kc * TC_KC + 4 * kg + kk;
      const float2 v = raw[((om >> 4) * FO + i) * int64_t(f) * 16 + int64_t(j) * 16 + (om & 15)];
      re[kk] = v.x;
      im[kk] = v.y;
    }
    uint8_t* item = out + ((p * 2 + h) * nch + kc) * int64_t(C::WITEM);
#pragma unroll
    for (int blk = 0; blk < 3; ++blk) {
      float hv[4], lv[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const float x = blk == 0 ? -im[kk] : blk == 1 ? re[kk] : im[kk];
        split_tf32(x, hv[kk], lv[kk]);
      }
      const int off = tile_off(blk * C::NS + n, kg);
      *reinterpret_cast<float4*>(item + (w * 2 + 0) * C::BMAT + off) = make_float4(hv[0], hv[1], hv[2], hv[3]);
      if constexpr (BFC) {
        // bf16 correction matrix (K = 16): K 0-7 = bf16(lo), K 8-15 = bf16(hi) of the
        // 8 channels; this thread's 4 channels are 8 bytes of each 16-byte K group
        uint8_t* cm = item + (w * 2 + 1) * C::BMAT + tile_off(blk * C::NS + n, 0) + 8 * kg;
        *reinterpret_cast<uint2*>(cm) = make_uint2(pack_bf16(lv[0], lv[1]), pack_bf16(lv[2], lv[3]));
        *reinterpret_cast<uint2*>(cm + 128) = make_uint2(pack_bf16(hv[0], hv[1]), pack_bf16(hv[2], hv[3]));
      } else {
        *reinterpret_cast<float4*>(item + (w * 2 + 1) * C::BMAT + off) = make_float4(lv[0], lv[1], lv[2], lv[3]);
      }
    }
  }
}

__device__ __forceinline__ void st_global_v8(void* p, float4 a, float4 b) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"l"(p), "f"(a.x), "f"(a.y), "f"(a.z),
               "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
               : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(addr));
}

struct QArgs {
  float2* Y;
  const uint8_t* W;
  int64_t M, mstride;
  int f, fo, mblocks;
  int64_t nwb;
  int raw_bytes;    // bytes one X box lands in shared memory
  int dbg;          // VXG_TC_DBG experiment switches, results invalid when set:
                    // 2 skip the Y stores, 4 skip the epilogue's TMEM loads, 8 skip the A stores
  long long* prof;
};

// BFC: 2 MMAs per product instead of 3 -- a*b ~ a_hi*b_hi (tf32) + [bf16(a_hi) |
// bf16(a_lo)] . [bf16(b_lo) ; bf16(b_hi)] (one kind::f16 MMA, K = 16): the
// correction terms are ~2^-11 of the product, so their bf16 rounding costs
// ~2^-19 relative per product (3xTF32: ~2^-21).
template <int FO, bool BFC>
__global__ void __launch_bounds__(Q_THREADS, 1)
    cgemm_q_kernel(const __grid_constant__ CUtensorMap xmap, QArgs a) {
  using C = QCfg<FO>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* rfull = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);  // [RS] X box landed (tx)
  uint64_t* rfree = rfull + C::RS;         // [RS] X box read by the converters
  uint64_t* wfull = rfree + C::RS;         // [AS] W item landed (tx)
  uint64_t* ready = wfull + C::AS;         // [AS] A slot written (converters)
  uint64_t* aempty = ready + C::AS;        // [AS] A slot and W slot consumed (MMA commit)
  uint64_t* acc_full = aempty + C::AS;     // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = a.f / TC_KC;
  const int64_t ntiles = a.nwb * a.mblocks * 8;
  const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t nitems = my_tiles * 2 * nch;  // items (tile, pass, chunk)

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 32) {
    for (int s = 0; s < C::RS; ++s) {
      mbar_init(&rfull[s], 1);    // X producer's arrive + transaction bytes
      mbar_init(&rfree[s], 128);  // converter threads (one group per item)
    }
    for (int s = 0; s < C::AS; ++s) {
      mbar_init(&wfull[s], 1);    // W producer's arrive + transaction bytes
      mbar_init(&ready[s], 128);  // converter threads (one group per item)
      mbar_init(&aempty[s], 1);   // MMA commit
    }
    for (int p = 0; p < 2; ++p) {
      mbar_init(&acc_full[p], 1);
      mbar_init(&acc_empty[p], 128);  // epilogue threads
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_slot;

  // tile t (local) -> (line block wb, row block, quad q, half h), (q, h) fastest
  // (grouping row blocks so fewer CTAs share a W item at a time made no
  // difference, profiles/r2_experiments.md §7)
  auto tile_of = [&](int64_t lt, int64_t& wb, int64_t& m0, int& q, int& h) {
    const int64_t t = blockIdx.x + lt * gridDim.x;
    h = int(t & 1);
    q = int((t >> 1) & 3);
    const int64_t rest = t >> 3;
    m0 = (rest % a.mblocks) * TC_M;
    wb = rest / a.mblocks;
  };

  if (warp == 0 || warp == 2) {
    // ---------------- producers (one thread each): X boxes (warp 0), W items (warp 2) ----------------
    if (lane == 0) {
      const bool xp = warp == 0;
      long long pw = 0;
      // running ring position (no 64-bit divisions in the item loop)
      int s = 0;
      uint32_t ph = 0;
      bool wrapped = false;
      const int depth = xp ? C::RS : C::AS;
      for (int64_t t = 0; t < my_tiles; ++t) {
        int64_t wb, m0;
        int q, h;
        tile_of(t, wb, m0, q, h);
        for (int pass = 0; pass < 2; ++pass)
          for (int kc = 0; kc < nch; ++kc) {
            const long long t0 = a.prof ? clock64() : 0;
            if (wrapped) mbar_wait(xp ? &rfree[s] : &aempty[s], ph ^ 1u);
            if (a.prof) pw += clock64() - t0;
            if (xp) {
              // X: floats [q*8 + pass*4, +4) of the 8 channel lines from kc*8, 128 rows
              mbar_arrive_expect_tx(&rfull[s], a.raw_bytes);
              for (int ch = 0; ch < TC_KC; ++ch)
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                    "[%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(smem + s * Q_RAW + ch * TC_M * 16)),
                    "l"(&xmap), "r"(q * 8 + pass * 4), "r"(kc * TC_KC + ch), "r"(int(m0)), "r"(int(wb)),
                    "r"(smem_u32(&rfull[s]))
                    : "memory");
            } else {
              const int64_t pair = wb * 8 + q * 2 + pass;
              mbar_arrive_expect_tx(&wfull[s], C::WITEM);
              bulk_copy(smem + C::OFF_W + s * C::WITEM,
                        a.W + ((pair * 2 + h) * nch + kc) * int64_t(C::WITEM), C::WITEM, &wfull[s]);
            }
            if (++s == depth) {
              s = 0;
              ph ^= 1u;
              wrapped = true;
            }
          }
      }
      if (a.prof && xp) a.prof[blockIdx.x * 8 + 0] = pw;
    }
  } else if (warp >= 8) {
    // ---------------- converters: thread c owns row c ----------------
    // two converter groups, each a thread per row: warps 8-11 take the even
    // items, warps 12-15 the odd ones, so two items' TMEM stores are in flight
    const int c = (tid - 256) & 127;
    const int grp = (tid - 256) >> 7;
    long long cw = 0, cb = 0;
    int s = grp, as = grp;
    uint32_t ph = 0, aph = 0;
    for (int64_t g = grp; g < nitems; g += 2) {
      const long long t0 = a.prof ? clock64() : 0;
      mbar_wait(&rfull[s], ph);
      long long t1 = a.prof ? clock64() : 0;
      cw += t1 - t0;
      const uint8_t* raw = smem + s * Q_RAW + c * 16;
      // split X row c into tf32 hi/lo: A slot columns ((w*2 + comp)*2 + hi/lo)*8 + channel
      // (BFC: the lo part's 8 columns hold the packed bf16 correction operand:
      // columns 0-3 bf16(hi) of channels (0,1)..(6,7), columns 4-7 bf16(lo))
      uint32_t u[64];
      float2 hl[4][8];
      (void)hl;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const float4 v = *reinterpret_cast<const float4*>(raw + ch * (TC_M * 16));  // (re0, im0, re1, im1)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float x = e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
          float hi, lo;
          split_tf32(x, hi, lo);
          u[(e * 2 + 0) * 8 + ch] = __float_as_uint(hi);
          if constexpr (!BFC) u[(e * 2 + 1) * 8 + ch] = __float_as_uint(lo);
          else hl[e][ch] = make_float2(hi, lo);
        }
      }
      if constexpr (BFC) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int c2 = 0; c2 < 4; ++c2) {
            u[(e * 2 + 1) * 8 + c2] = pack_bf16(hl[e][2 * c2].x, hl[e][2 * c2 + 1].x);
            u[(e * 2 + 1) * 8 + 4 + c2] = pack_bf16(hl[e][2 * c2].y, hl[e][2 * c2 + 1].y);
          }
      }
      // the box may be refilled: order these generic-proxy reads before the
      // producer's next TMA (async-proxy) write into the slot
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // required: without it the refill races the reads
      mbar_arrive(&rfree[s]);
      if (a.prof) cb += clock64() - t1;
      t1 = a.prof ? clock64() : 0;
      if (g >= C::AS) mbar_wait(&aempty[as], aph ^ 1u);  // the MMAs reading this A slot are done
      if (a.prof) {
        const long long t2 = clock64();
        cw += t2 - t1;
        t1 = t2;
      }
      const uint32_t ta = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(C::ACOL + 64 * as);
      if (!(a.dbg & 8)) asm volatile(
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
      mbar_arrive(&ready[as]);
      if (a.prof) cb += clock64() - t1;
      // both rings advance by two items per group step
      s += 2;
      if (s >= C::RS) {
        s -= C::RS;
        ph ^= 1u;
      }
      as += 2;
      if (as >= C::AS) {
        as -= C::AS;
        aph ^= 1u;
      }
    }
    if (a.prof && c == 0 && grp == 0) {
      a.prof[blockIdx.x * 8 + 1] = cw;
      a.prof[blockIdx.x * 8 + 2] = cb;
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      long long me = 0, mr = 0;
      const long long tstart = a.prof ? clock64() : 0;
      const uint32_t idesc = idesc_tf32<FO>(false);
      int as = 0;
      uint32_t aph = 0;
      for (int64_t t = 0; t < my_tiles; ++t)
        for (int pass = 0; pass < 2; ++pass)
          for (int kc = 0; kc < nch; ++kc) {
        const long long t0 = a.prof ? clock64() : 0;
        if (kc == 0 && t > 0) mbar_wait(&acc_empty[pass], uint32_t((t - 1) & 1));  // pass drained
        const long long t1 = a.prof ? clock64() : 0;
        mbar_wait(&ready[as], aph);
        mbar_wait(&wfull[as], aph);
        if (a.prof) {
          me += t1 - t0;
          mr += clock64() - t1;
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const uint32_t wbase = smem_u32(smem + C::OFF_W + as * C::WITEM);
        const uint32_t ta = tmem + uint32_t(C::ACOL + 64 * as);
        const uint32_t acc0 = kc > 0 ? 1u : 0u;
        // (A comp, A hi/lo, B block start, B hi/lo): Xr [Wr | Wi] + Xi [-Wi | Wr],
        // ordered so consecutive MMAs share their B matrix where they can
        constexpr int TERMS[6][4] = {{0, 0, 1, 0}, {0, 1, 1, 0}, {0, 0, 1, 1},
                                     {1, 0, 0, 1}, {1, 0, 0, 0}, {1, 1, 0, 0}};
        auto issue = [&](int w, int k) {
          const uint32_t d = tmem + uint32_t((pass * 2 + w) * FO);
          const uint32_t am = ta + uint32_t(((w * 2 + TERMS[k][0]) * 2 + TERMS[k][1]) * 8);
          const uint64_t bm = umma_desc(wbase + (w * 2 + TERMS[k][3]) * C::BMAT + TERMS[k][2] * (NS / 8) * 256);
          mma_tf32_ta(d, am, bm, idesc, k == 0 ? acc0 : 1u);
        };
        if constexpr (BFC) {
          // per frequency: Xr_hi [Wr|Wi]_hi, Xr_corr [Wr|Wi]_corr, Xi_hi [-Wi|Wr]_hi, Xi_corr [-Wi|Wr]_corr
          const uint32_t idb = idesc_bf16<FO>();
#pragma unroll
          for (int w = 0; w < 2; ++w)
#pragma unroll
            for (int comp = 0; comp < 2; ++comp) {
              const uint32_t d = tmem + uint32_t((pass * 2 + w) * FO);
              const int blk = comp == 0 ? 1 : 0;  // B_top starts at block 1, B_bot at block 0
              const uint32_t bb = wbase + blk * (NS / 8) * 256;
              mma_tf32_ta(d, ta + uint32_t(((w * 2 + comp) * 2 + 0) * 8), umma_desc(bb + (w * 2 + 0) * C::BMAT), idesc,
                          comp == 0 ? acc0 : 1u);
              mma_bf16_ta(d, ta + uint32_t(((w * 2 + comp) * 2 + 1) * 8), umma_desc(bb + (w * 2 + 1) * C::BMAT), idb,
                          1u);
            }
        } else {
#pragma unroll
          for (int w = 0; w < 2; ++w)
#pragma unroll
            for (int k = 0; k < 6; ++k) issue(w, k);
        }
        (void)issue;
        umma_commit(&aempty[as]);                        // A slot and W slot reusable once these MMAs finish
        if (kc == nch - 1) umma_commit(&acc_full[pass]);  // pass accumulated
        if (++as == C::AS) {
          as = 0;
          aph ^= 1u;
        }
          }
      if (a.prof) {
        a.prof[blockIdx.x * 8 + 3] = me;
        a.prof[blockIdx.x * 8 + 4] = mr;
        a.prof[blockIdx.x * 8 + 7] = clock64() - tstart;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: warp 4+qd owns TMEM lanes 32qd .. 32qd+31 ----------------
    const int qd = warp - 4;
    const int row = qd * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t(qd * 32) << 16);
    uint8_t* park = smem + C::OFF_PARK + row * C::PARK_ROW;
    long long ew = 0, eb = 0;
    for (int64_t t = 0; t < my_tiles; ++t) {
      int64_t wb, m0;
      int q, h;
      tile_of(t, wb, m0, q, h);
      const int64_t m = m0 + row;
      // pass 0: frequencies 4q, 4q+1 -> park (re0, im0, re1, im1) per map
      long long t0 = a.prof ? clock64() : 0;
      mbar_wait(&acc_full[0], uint32_t(t & 1));
      long long t1 = a.prof ? clock64() : 0;
      ew += t1 - t0;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
#pragma unroll 1
      for (int i0 = 0; i0 < ((a.dbg & 4) ? 0 : NS); i0 += 8) {
        uint32_t r0[8], i0v[8], r1[8], i1v[8];
        tmem_ld8(lane_base + uint32_t(0 * FO + i0), r0);
        tmem_ld8(lane_base + uint32_t(0 * FO + NS + i0), i0v);
        tmem_ld8(lane_base + uint32_t(1 * FO + i0), r1);
        tmem_ld8(lane_base + uint32_t(1 * FO + NS + i0), i1v);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
#pragma unroll
        for (int ii = 0; ii < 8; ++ii)
          *reinterpret_cast<float4*>(park + (i0 + ii) * 16) =
              make_float4(__uint_as_float(r0[ii]), __uint_as_float(i0v[ii]), __uint_as_float(r1[ii]),
                          __uint_as_float(i1v[ii]));
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(&acc_empty[0]);
      if (a.prof) eb += clock64() - t1;
      // pass 1: frequencies 4q+2, 4q+3 -> whole 32-byte sectors
      t0 = a.prof ? clock64() : 0;
      mbar_wait(&acc_full[1], uint32_t(t & 1));
      t1 = a.prof ? clock64() : 0;
      ew += t1 - t0;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      float2* yrow = a.Y + ((wb * a.mstride + m) * a.fo + h * NS) * 16 + q * 4;
#pragma unroll 1
      for (int i0 = 0; i0 < ((a.dbg & 4) ? 0 : NS); i0 += 8) {
        uint32_t r2[8], i2v[8], r3[8], i3v[8];
        tmem_ld8(lane_base + uint32_t(2 * FO + i0), r2);
        tmem_ld8(lane_base + uint32_t(2 * FO + NS + i0), i2v);
        tmem_ld8(lane_base + uint32_t(3 * FO + i0), r3);
        tmem_ld8(lane_base + uint32_t(3 * FO + NS + i0), i3v);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
        if (m < a.M && !(a.dbg & 2)) {
#pragma unroll
          for (int ii = 0; ii < 8; ++ii) {
            const float4 lo = *reinterpret_cast<const float4*>(park + (i0 + ii) * 16);
            st_global_v8(yrow + (i0 + ii) * 16, lo,
                         make_float4(__uint_as_float(r2[ii]), __uint_as_float(i2v[ii]), __uint_as_float(r3[ii]),
                                     __uint_as_float(i3v[ii])));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      mbar_arrive(&acc_empty[1]);
      if (a.prof) eb += clock64() - t1;
    }
    if (a.prof && qd == 0 && lane == 0) {
      a.prof[blockIdx.x * 8 + 5] = ew;
      a.prof[blockIdx.x * 8 + 6] = eb;
    }
  }
  // warp 3 and lanes 1-31 of warps 0-2 have no role
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}


template <int FO>
void q_t(Ctx* c, const GemmArgs& g, int64_t npairs) {
  using C = QCfg<FO>;
  static_assert(C::SMEM <= 232448, "cgemm_q: shared memory");
  static PerDeviceOnce configured;
  if (configured.first()) {
    VXG_CUDA_CHECK(cudaFuncSetAttribute(cgemm_q_kernel<FO, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    VXG_CUDA_CHECK(cudaFuncSetAttribute(cgemm_q_kernel<FO, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  }
  QArgs a{};
  a.Y = g.Y;
  a.W = reinterpret_cast<const uint8_t*>(g.W);
  a.M = g.M;
  a.mstride = g.mstride;
  a.f = g.f;
  a.fo = g.fo;
  a.mblocks = int((g.M + TC_M - 1) / TC_M);
  a.nwb = npairs / 8;
  // X as a 4D f32 tensor: (32 floats of a line, channel, row, line block)
  CUtensorMap xmap;
  const uint64_t dims[4] = {32, uint64_t(g.f), uint64_t(g.mstride), uint64_t(a.nwb)};
  const uint64_t strides[3] = {128, uint64_t(g.f) * 128, uint64_t(g.mstride) * g.f * 128};
  // one box per channel line: 4 floats x 128 rows (fewer rows when the layer
  // is that small: a box may not exceed the tensor)
  const uint32_t brows = uint32_t(std::min<int64_t>(TC_M, g.mstride));
  const uint32_t box[4] = {4, 1, brows, 1};
  a.raw_bytes = int(16 * TC_KC * brows);
  static const int dbg = std::getenv("VXG_TC_DBG") ? std::atoi(std::getenv("VXG_TC_DBG")) : 0;
  a.dbg = dbg;
  encode_tensor_map_f32(&xmap, g.X, 4, dims, strides, box);
  const int64_t ntiles = a.nwb * a.mblocks * 8;
  const unsigned grid = unsigned(std::min<int64_t>(ntiles, c->num_sms));
  static const bool prof = std::getenv("VXG_TC_PROF") != nullptr;
  long long* dprof = nullptr;
  if (prof) {
    VXG_CUDA_CHECK(cudaMalloc(&dprof, size_t(grid) * 8 * sizeof(long long)));
    VXG_CUDA_CHECK(cudaMemset(dprof, 0, size_t(grid) * 8 * sizeof(long long)));
    a.prof = dprof;
  }
  if (q_bf16_correction())
    cgemm_q_kernel<FO, true><<<grid, Q_THREADS, C::SMEM, c->stream>>>(xmap, a);
  else
    cgemm_q_kernel<FO, false><<<grid, Q_THREADS, C::SMEM, c->stream>>>(xmap, a);
  c->counted();
  check_launch("cgemm_q_kernel");
  if (prof) {
    std::vector<long long> h(size_t(grid) * 8);
    VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    VXG_CUDA_CHECK(cudaMemcpy(h.data(), dprof, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(dprof);
    double mm[8] = {0};
    for (unsigned b = 0; b < grid; ++b)
      for (int k = 0; k < 8; ++k) mm[k] += double(h[b * 8 + k]) / grid;
    std::fprintf(stderr,
                 "[qprof] M=%lld total %.3gM | producer wait %.3gM | converter wait %.3gM busy %.3gM | "
                 "mma wait-epilogue %.3gM wait-ready %.3gM | epilogue wait %.3gM busy %.3gM\n",
                 (long long)g.M, mm[7] / 1e6, mm[0] / 1e6, mm[1] / 1e6, mm[2] / 1e6, mm[3] / 1e6, mm[4] / 1e6,
                 mm[5] / 1e6, mm[6] / 1e6);
  }
}

template <int FO>
void q_wsplit_t(Ctx* c, const float2* raw, void* out, int64_t npairs, int f) {
  using C = QCfg<FO>;
  const int64_t total = npairs * 2 * (f / TC_KC) * 2 * C::NS * 2;
  if (q_bf16_correction())
    q_wsplit_kernel<FO, true><<<grid_for(total, 256, int64_t(c->num_sms) * 16), 256, 0, c->stream>>>(
        raw, static_cast<uint8_t*>(out), npairs, f);
  else
    q_wsplit_kernel<FO, false><<<grid_for(total, 256, int64_t(c->num_sms) * 16), 256, 0, c->stream>>>(
        raw, static_cast<uint8_t*>(out), npairs, f);
  c->counted();
  check_launch("q_wsplit_kernel");
}

}  // namespace

// VXG_TC_PAIR=1 keeps the pair-tile kernel (cgemm_tc_kernel) for A/B timing;
// the pair-major Y experiment (VXG_YPAIR=1) needs it too
bool tc_quad_enabled() {
  const char* e = std::getenv("VXG_TC_PAIR");
  const char* y = std::getenv("VXG_YPAIR");
  return !(e && std::strcmp(e, "0") != 0) && !(y && std::strcmp(y, "1") == 0);
}

int64_t q_wsplit_bytes(int64_t npairs, int64_t f, int64_t fo) {
  // per (pair, half, chunk): 2 frequencies x hi/lo x 3 blocks x (fo/2) x 8 tf32
  return npairs * 2 * (f / TC_KC) * 4 * 3 * (fo / 2) * TC_KC * 4;
}

#define VXG_Q_SWITCH(CALL)                                            \
  switch (fo) {                                                       \
    case 16: CALL(16); break;                                         \
    case 32: CALL(32); break;                                         \
    case 48: CALL(48); break;                                         \
    case 64: CALL(64); break;                                         \
    case 80: CALL(80); break;                                         \
    default: throw invalid("cgemm_q: unsupported output map count"); \
  }

void q_wsplit(Ctx* c, const float2* raw, void* out, int64_t npairs, int64_t f, int64_t fo) {
  KScope ks(c, VXG_K_KSPEC, 0.0, double(npairs) * 2 * f * fo * (16.0 + 24.0));
#define VXG_QW(F) q_wsplit_t<F>(c, raw, out, npairs, int(f))
  VXG_Q_SWITCH(VXG_QW)
#undef VXG_QW
}

void launch_cgemm_q(Ctx* c, const GemmArgs& a, int64_t npairs) {
  const double nw = double(a.T) * a.T * (a.T / 2 + 1);
  KScope ks(c, VXG_K_CGEMM, 8.0 * double(a.M) * a.f * a.fo * nw,
            8.0 * nw * (double(a.M) * a.f + double(a.M) * a.fo + double(a.f) * a.fo));
  const int64_t fo = a.fo;
#define VXG_Q(F) q_t<F>(c, a, npairs)
  VXG_Q_SWITCH(VXG_Q)
#undef VXG_Q
}

}  // namespace vxg
