// K3 on CTA pairs (tcgen05 cta_group::2): the quad-frequency contraction of
// k_cgemm_q.cu with M = 256 rows per MMA, split over the two SMs of a pair.
//
// Same math and product scheme as k_cgemm_q.cu (per real product a tf32 MMA
// for a_hi*b_hi plus one bf16 kind::f16 correction MMA, K = 16), same tile
// (4 consecutive frequencies x half the output maps, two passes of 2
// frequencies, whole 32-byte sector stores), but one MMA instruction now
// covers 256 rows: each CTA of the pair converts its own 128 rows of X into
// its own TMEM A slot and holds its own 128 x fo accumulators, and the B
// operand -- the real-block kernel spectra -- is split by columns between the
// two CTAs' shared memory:
//     [Dr | Di] += Xr [Wr | Wi] + Xi [-Wi | Wr]
//     CTA 0 holds (slot A, slot B) = (Wr, -Wi), CTA 1 holds (Wi, Wr).
// So each CTA stages 2 NS x 8 blocks per (frequency, part) instead of the
// single-CTA kernel's 3, for twice the rows: the kernel-spectrum stream
// through L2 drops to 1/3 per row (it was ~37 % of the kernel's L2 traffic,
// the resource the single-CTA kernel is bound by), and the MMA issuer issues
// half the instructions per row.
//
// Pipeline (per CTA, mbarrier handshakes; the leader CTA, rank 0, issues all MMAs):
//   warp 0 lane 0  X producer: one TMA box per item (its 128 rows, the pass's
//                  16-byte piece of 8 channel lines, 128-byte swizzle) into a
//                  ring freed by the converters;
//   warp 2 lane 0  W producer: one bulk copy of this CTA's half of the item's
//                  pre-split W into a ring shared with the TMEM A slots;
//   warp 3 lane 0  (rank 1) forwards "W landed" to the leader;
//   warps 8-15     converters (two groups, alternate items): split X into
//                  tf32 hi / bf16 correction, tcgen05.st into the A slot,
//                  arrive on the LEADER's ready barrier;
//   warp 1 lane 0  (rank 0) MMA issuer: waits for both CTAs' A slots and W
//                  halves, 8 cta_group::2 MMAs per item, commits multicast to
//                  both CTAs (slot free; pass accumulated);
//   warps 4-7      epilogue (its own TMEM), arrive on the leader's acc_empty.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "fftconv.hpp"
#include "tcgen05.cuh"

namespace vxg {

void encode_tensor_map_f32(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
                           const uint64_t* strides, const uint32_t* box, bool swizzle128);

// VXG_Q2=1: CTA pairs instead of the single-CTA quad kernel (k_cgemm_q.cu)
// (the W layout follows the same switch; 3xTF32 runs single-CTA only)
bool q2_enabled() {
  const char* e = std::getenv("VXG_Q2");
  return e && std::strcmp(e, "1") == 0 && q_bf16_correction();
}

namespace {

using namespace tc;
constexpr int Q2_THREADS = 512;
constexpr int Q2_RAW = TC_M * 128;  // swizzled X box: 128 rows x 8 pieces of 16 B

template <int FO>
struct Q2Cfg {
  static constexpr int AS = 4 * FO + 4 * 64 <= 512 ? 4 : 3;
  static constexpr int NS = FO / 2;
  static constexpr int BM = NS * TC_KC * 4;        // one NS x 8 block (tf32, or bf16 K = 16)
  static constexpr int WHALF = 8 * BM;             // one CTA's share of an item: (w, part, slot)
  static constexpr int WITEM = 2 * WHALF;          // both CTAs
  static constexpr int PARK_ROW = NS * 16 + 16;
  static constexpr int BAR_BYTES = 512;
  static constexpr int RS_FIT = (232448 - BAR_BYTES - TC_M * PARK_ROW - AS * WHALF) / Q2_RAW;
  static constexpr int RS = RS_FIT > 8 ? 8 : RS_FIT;
  static constexpr int OFF_W = RS * Q2_RAW;
  static constexpr int OFF_PARK = OFF_W + AS * WHALF;
  static constexpr int OFF_BAR = OFF_PARK + TC_M * PARK_ROW;
  static constexpr int SMEM = OFF_BAR + BAR_BYTES;
  static constexpr int ACOL = 4 * FO;
  static_assert((2 * RS + 4 * AS + 4) * 8 + 4 <= BAR_BYTES, "cgemm_q2: barrier area");
  static_assert(Q2_RAW % 1024 == 0, "cgemm_q2: swizzled ring slots must be 1024-byte aligned");
};

// M = 256 (cta_group::2), N = FO
template <int N>
__device__ __forceinline__ constexpr uint32_t idesc2_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(256 >> 4) << 24);
}
template <int N>
__device__ __forceinline__ constexpr uint32_t idesc2_bf16() {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(256 >> 4) << 24);
}

__device__ __forceinline__ void mma2_tf32_ta(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma2_bf16_ta(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
// arrive on the same barrier offset in both CTAs once the issued MMAs finish
__device__ __forceinline__ void umma_commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<unsigned short>(3))
      : "memory");
}
__device__ __forceinline__ uint32_t leader_addr(const void* local) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(r) : "r"(smem_u32(local)));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
// wait on a barrier that receives arrivals from the other CTA
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cta_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

// raw [w/16][i][j][16] complex -> per item (pair p, half h, chunk kc), per CTA
// r, per (frequency w, part hi/corr, slot A/B) one NS x 8 block in the UMMA
// K-major layout: r = 0 (Wr, -Wi), r = 1 (Wi, Wr)
template <int FO>
__global__ void q2_wsplit_kernel(const float2* __restrict__ raw, uint8_t* __restrict__ out, int64_t npairs,
                                 int f) {
  using C = Q2Cfg<FO>;
  const int nch = f / TC_KC;
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
    const int64_t om = 2 * p + w;
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
    for (int rk = 0; rk < 2; ++rk)
#pragma unroll
      for (int slot = 0; slot < 2; ++slot) {
        float hv[4], lv[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float x = rk == 0 ? (slot == 0 ? re[kk] : -im[kk]) : (slot == 0 ? im[kk] : re[kk]);
          split_tf32(x, hv[kk], lv[kk]);
        }
        uint8_t* hb = item + rk * C::WHALF + ((w * 2 + 0) * 2 + slot) * C::BM;
        uint8_t* cb = item + rk * C::WHALF + ((w * 2 + 1) * 2 + slot) * C::BM;
        *reinterpret_cast<float4*>(hb + tile_off(n, kg)) = make_float4(hv[0], hv[1], hv[2], hv[3]);
        // bf16 correction (K = 16): K 0-7 bf16(lo), K 8-15 bf16(hi) of the 8 channels
        uint8_t* cm = cb + tile_off(n, 0) + 8 * kg;
        *reinterpret_cast<uint2*>(cm) = make_uint2(pack_bf16(lv[0], lv[1]), pack_bf16(lv[2], lv[3]));
        *reinterpret_cast<uint2*>(cm + 128) = make_uint2(pack_bf16(hv[0], hv[1]), pack_bf16(hv[2], hv[3]));
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

struct Q2Args {
  float2* Y;
  const uint8_t* W;
  int64_t M, mstride;
  int f, fo, mblocks2;  // 256-row blocks
  int64_t nwb;
  int raw_bytes;
};

template <int FO>
__global__ void __launch_bounds__(Q2_THREADS, 1)
    cgemm_q2_kernel(const __grid_constant__ CUtensorMap xmap, Q2Args a) {
  using C = Q2Cfg<FO>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* rfull = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);  // [RS] X box landed (tx)
  uint64_t* rfree = rfull + C::RS;       // [RS] X box read by the converters
  uint64_t* wfull = rfree + C::RS;       // [AS] this CTA's W half landed (tx)
  uint64_t* wpeer = wfull + C::AS;       // [AS] leader: the peer's W half landed
  uint64_t* ready = wpeer + C::AS;       // [AS] leader: both CTAs' A slots written (256)
  uint64_t* aempty = ready + C::AS;      // [AS] A and W slots consumed (multicast commit)
  uint64_t* acc_full = aempty + C::AS;   // [2] pass accumulated (multicast commit)
  uint64_t* acc_empty = acc_full + 2;    // [2] leader: both epilogues drained the pass (256)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const unsigned rank = cta_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = a.f / TC_KC;
  const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int64_t ntiles = a.nwb * a.mblocks2 * 8;
  const int64_t my_tiles = (ntiles - cid + ncl - 1) / ncl;
  const int64_t nitems = my_tiles * 2 * nch;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  if (tid == 32) {
    for (int s = 0; s < C::RS; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rfree[s], 128);
    }
    for (int s = 0; s < C::AS; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wpeer[s], 1);
      mbar_init(&ready[s], 256);
      mbar_init(&aempty[s], 1);
    }
    for (int p = 0; p < 2; ++p) {
      mbar_init(&acc_full[p], 1);
      mbar_init(&acc_empty[p], 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_slot;

  // pair tile t -> (line block wb, 256-row block, quad q, half h); this CTA's rows m0 ..
  auto tile_of = [&](int64_t lt, int64_t& wb, int64_t& m0, int& q, int& h) {
    const int64_t t = cid + lt * ncl;
    h = int(t & 1);
    q = int((t >> 1) & 3);
    const int64_t rest = t >> 3;
    m0 = (rest % a.mblocks2) * (2 * TC_M) + int64_t(rank) * TC_M;
    wb = rest / a.mblocks2;
  };

  if (warp == 0 || warp == 2) {
    if (lane == 0) {
      const bool xp = warp == 0;
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
            if (wrapped) mbar_wait(xp ? &rfree[s] : &aempty[s], ph ^ 1u);
            if (xp) {
              mbar_arrive_expect_tx(&rfull[s], a.raw_bytes);
              asm volatile(
                  "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                  "[%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(smem + s * Q2_RAW)),
                  "l"(&xmap), "r"(q * 8 + pass * 4), "r"(kc * TC_KC), "r"(int(m0)), "r"(int(wb)),
                  "r"(smem_u32(&rfull[s]))
                  : "memory");
            } else {
              const int64_t pair = wb * 8 + q * 2 + pass;
              mbar_arrive_expect_tx(&wfull[s], C::WHALF);
              bulk_copy(smem + C::OFF_W + s * C::WHALF,
                        a.W + ((pair * 2 + h) * nch + kc) * int64_t(C::WITEM) + int64_t(rank) * C::WHALF,
                        C::WHALF, &wfull[s]);
            }
            if (++s == depth) {
              s = 0;
              ph ^= 1u;
              wrapped = true;
            }
          }
      }
    }
  } else if (warp == 3) {
    // rank 1: tell the leader when this CTA's W half of each item has landed
    if (rank == 1 && lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t g = 0; g < nitems; ++g) {
        mbar_wait(&wfull[s], ph);
        mbar_arrive_remote(leader_addr(&wpeer[s]));
        if (++s == C::AS) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp >= 8) {
    // ---------------- converters: thread c owns row c of this CTA ----------------
    const int c = (tid - 256) & 127;
    const int grp = (tid - 256) >> 7;
    const int sw = c & 7;  // swizzled staged row: piece ch at 16 * (ch ^ (c & 7))
    int s = grp, as = grp;
    uint32_t ph = 0, aph = 0;
    for (int64_t g = grp; g < nitems; g += 2) {
      mbar_wait(&rfull[s], ph);
      const uint8_t* rawp = smem + s * Q2_RAW + c * 128;
      uint32_t u[64];
      float2 hl[4][8];
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const float4 v = *reinterpret_cast<const float4*>(rawp + (ch ^ sw) * 16);  // (re0, im0, re1, im1)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float x = e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
          float hi, lo;
          split_tf32(x, hi, lo);
          u[(e * 2 + 0) * 8 + ch] = __float_as_uint(hi);
          hl[e][ch] = make_float2(hi, lo);
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int c2 = 0; c2 < 4; ++c2) {
          u[(e * 2 + 1) * 8 + c2] = pack_bf16(hl[e][2 * c2].x, hl[e][2 * c2 + 1].x);
          u[(e * 2 + 1) * 8 + 4 + c2] = pack_bf16(hl[e][2 * c2].y, hl[e][2 * c2 + 1].y);
        }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // reads before the TMA refill
      mbar_arrive(&rfree[s]);
      if (g >= C::AS) mbar_wait(&aempty[as], aph ^ 1u);
      const uint32_t ta = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(C::ACOL + 64 * as);
      asm volatile(
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
      mbar_arrive_remote(leader_addr(&ready[as]));
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
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    if (rank == 0 && lane == 0) {
      const uint32_t idt = idesc2_tf32<FO>();
      const uint32_t idb = idesc2_bf16<FO>();
      int as = 0;
      uint32_t aph = 0;
      for (int64_t t = 0; t < my_tiles; ++t)
        for (int pass = 0; pass < 2; ++pass)
          for (int kc = 0; kc < nch; ++kc) {
            if (kc == 0 && t > 0) mbar_wait_cl(&acc_empty[pass], uint32_t((t - 1) & 1));
            mbar_wait_cl(&ready[as], aph);
            mbar_wait(&wfull[as], aph);
            mbar_wait_cl(&wpeer[as], aph);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
            const uint32_t wbase = smem_u32(smem + C::OFF_W + as * C::WHALF);
            const uint32_t ta = tmem + uint32_t(C::ACOL + 64 * as);
            const uint32_t acc0 = kc > 0 ? 1u : 0u;
#pragma unroll
            for (int w = 0; w < 2; ++w)
#pragma unroll
              for (int comp = 0; comp < 2; ++comp) {
                // comp 0: Xr . slot A ([Wr | Wi]); comp 1: Xi . slot B ([-Wi | Wr])
                const uint32_t d = tmem + uint32_t((pass * 2 + w) * FO);
                mma2_tf32_ta(d, ta + uint32_t(((w * 2 + comp) * 2 + 0) * 8),
                             umma_desc(wbase + ((w * 2 + 0) * 2 + comp) * C::BM), idt, comp == 0 ? acc0 : 1u);
                mma2_bf16_ta(d, ta + uint32_t(((w * 2 + comp) * 2 + 1) * 8),
                             umma_desc(wbase + ((w * 2 + 1) * 2 + comp) * C::BM), idb, 1u);
              }
            umma_commit2(&aempty[as]);
            if (kc == nch - 1) umma_commit2(&acc_full[pass]);
            if (++as == C::AS) {
              as = 0;
              aph ^= 1u;
            }
          }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: warp 4+qd owns TMEM lanes 32qd .. 32qd+31 ----------------
    const int qd = warp - 4;
    const int row = qd * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t(qd * 32) << 16);
    uint8_t* park = smem + C::OFF_PARK + row * C::PARK_ROW;
    const uint32_t empty0 = leader_addr(&acc_empty[0]), empty1 = leader_addr(&acc_empty[1]);
    for (int64_t t = 0; t < my_tiles; ++t) {
      int64_t wb, m0;
      int q, h;
      tile_of(t, wb, m0, q, h);
      const int64_t m = m0 + row;
      mbar_wait(&acc_full[0], uint32_t(t & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
#pragma unroll 1
      for (int i0 = 0; i0 < NS; i0 += 8) {
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
      mbar_arrive_remote(empty0);
      mbar_wait(&acc_full[1], uint32_t(t & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      float2* yrow = a.Y + ((wb * a.mstride + m) * a.fo + h * NS) * 16 + q * 4;
#pragma unroll 1
      for (int i0 = 0; i0 < NS; i0 += 8) {
        uint32_t r2[8], i2v[8], r3[8], i3v[8];
        tmem_ld8(lane_base + uint32_t(2 * FO + i0), r2);
        tmem_ld8(lane_base + uint32_t(2 * FO + NS + i0), i2v);
        tmem_ld8(lane_base + uint32_t(3 * FO + i0), r3);
        tmem_ld8(lane_base + uint32_t(3 * FO + NS + i0), i3v);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
        if (m < a.M) {
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
      mbar_arrive_remote(empty1);
    }
  }
  // both CTAs done (the leader's last MMAs read the peer's TMEM and signal its barriers)
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  cluster_sync_all();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

template <int FO>
void q2_t(Ctx* c, const GemmArgs& g, int64_t npairs) {
  using C = Q2Cfg<FO>;
  static_assert(C::SMEM <= 232448, "cgemm_q2: shared memory");
  static PerDeviceOnce configured;
  if (configured.first()) {
    VXG_CUDA_CHECK(cudaFuncSetAttribute(cgemm_q2_kernel<FO>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  }
  Q2Args a{};
  a.Y = g.Y;
  a.W = reinterpret_cast<const uint8_t*>(g.W);
  a.M = g.M;
  a.mstride = g.mstride;
  a.f = g.f;
  a.fo = g.fo;
  a.mblocks2 = int((g.M + 2 * TC_M - 1) / (2 * TC_M));
  a.nwb = npairs / 8;
  // X as a 4D f32 tensor (32 floats of a line, channel, row, line block); box:
  // the pass's 4 floats of 8 channel lines x 128 rows, 128-byte swizzle (rows
  // past mstride -- the second CTA of a short last block -- are zero-filled)
  CUtensorMap xmap;
  const uint64_t dims[4] = {32, uint64_t(g.f), uint64_t(g.mstride), uint64_t(a.nwb)};
  const uint64_t strides[3] = {128, uint64_t(g.f) * 128, uint64_t(g.mstride) * g.f * 128};
  // (a box may not exceed the tensor: fewer rows when the layer is that small)
  const uint32_t brows = uint32_t(std::min<int64_t>(TC_M, g.mstride));
  const uint32_t box[4] = {4, 8, brows, 1};
  a.raw_bytes = int(16 * 8 * brows);
  encode_tensor_map_f32(&xmap, g.X, 4, dims, strides, box, true);
  const int64_t ntiles = a.nwb * a.mblocks2 * 8;
  const int64_t pairs = std::min<int64_t>(ntiles, c->num_sms / 2);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(2 * pairs));
  cfg.blockDim = dim3(Q2_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  VXG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, cgemm_q2_kernel<FO>, xmap, a));
  c->counted();
  check_launch("cgemm_q2_kernel");
}

template <int FO>
void q2_wsplit_t(Ctx* c, const float2* raw, void* out, int64_t npairs, int f) {
  using C = Q2Cfg<FO>;
  const int64_t total = npairs * 2 * (f / TC_KC) * 2 * C::NS * 2;
  q2_wsplit_kernel<FO><<<grid_for(total, 256, int64_t(c->num_sms) * 16), 256, 0, c->stream>>>(
      raw, static_cast<uint8_t*>(out), npairs, f);
  c->counted();
  check_launch("q2_wsplit_kernel");
}

}  // namespace

int64_t q2_wsplit_bytes(int64_t npairs, int64_t f, int64_t fo) {
  // per (pair, half, chunk): 2 CTAs x 2 frequencies x (hi, corr) x 2 slots x (fo/2) x 8 x 4 B
  return npairs * 2 * (f / TC_KC) * 16 * (fo / 2) * TC_KC * 4;
}

#define VXG_Q2_SWITCH(CALL)                                            \
  switch (fo) {                                                        \
    case 16: CALL(16); break;                                          \
    case 32: CALL(32); break;                                          \
    case 48: CALL(48); break;                                          \
    case 64: CALL(64); break;                                          \
    case 80: CALL(80); break;                                          \
    default: throw invalid("cgemm_q2: unsupported output map count"); \
  }

void q2_wsplit(Ctx* c, const float2* raw, void* out, int64_t npairs, int64_t f, int64_t fo) {
  KScope ks(c, VXG_K_KSPEC, 0.0, double(npairs) * 2 * f * fo * (16.0 + 32.0));
#define VXG_QW2(F) q2_wsplit_t<F>(c, raw, out, npairs, int(f))
  VXG_Q2_SWITCH(VXG_QW2)
#undef VXG_QW2
}

void launch_cgemm_q2(Ctx* c, const GemmArgs& a, int64_t npairs) {
  const double nw = double(a.T) * a.T * (a.T / 2 + 1);
  KScope ks(c, VXG_K_CGEMM, 8.0 * double(a.M) * a.f * a.fo * nw,
            8.0 * nw * (double(a.M) * a.f + double(a.M) * a.fo + double(a.f) * a.fo));
  const int64_t fo = a.fo;
#define VXG_Q2(F) q2_t<F>(c, a, npairs)
  VXG_Q2_SWITCH(VXG_Q2)
#undef VXG_Q2
}

}  // namespace vxg
