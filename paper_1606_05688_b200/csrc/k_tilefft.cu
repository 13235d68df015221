// K1 / K2 / K4: on-chip tile transforms of the tiled pruned-FFT convolution.
//
// Math of conv_fft_data_parallel / conv_fft_staged / conv_fft_task_parallel
// (proj/include/voxin/layers.hpp:203-371, task_conv.hpp:415-442): valid
// convolution = crop of the circular convolution of zero-padded spectra.  The
// reference pads the WHOLE image to N(n) and multi-passes every axis through
// memory; here the output is cut into overlap-save tiles of a cubic FFT size
// T (T - k + 1 valid outputs per axis per tile), so that
//   * each 3D transform runs entirely on-chip: one HBM read of the tile box,
//     one write of its spectrum (K1 tile_fwd_kernel) and the reverse with the
//     crop, bias and ReLU fused into the store (K4 tile_inv_kernel, pruned to
//     the lines the crop needs, like pruned_inverse_region, fft.hpp:181-228);
//   * kernel spectra are small (T^3), computed once per layer by the same
//     forward kernel on the zero-filled k^3 kernels (K2) and pre-scaled by
//     1/T^3, so the inverse needs no normalisation pass.
// Spectra live in HBM as [w/16][row][channel][w%16] complex64 so every
// producer and consumer moves whole 128-byte lines; w = (kx*T + ky)*H + kz.
//
// Shared-memory layout: line (x, y) of z values lives in a slot of SY >= H
// complex (SY odd, so the slot-per-lane passes are bank-conflict free);
// x planes are SX apart with SX = H (mod 16) so the y-line pass is conflict
// free too.  One CTA owns one (tile, channel); every pass gives each thread
// exactly one register-resident line (THREADS = T*H rounded up to a warp).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "async.cuh"
#include "common.cuh"
#include "fft_reg.cuh"
#include "fftconv.hpp"

namespace vxg {

void init_twiddles() {
  std::vector<float2> h(fftreg::kTwTotal);
  for (int i = 0; i < fftreg::kNumSizes; ++i) {
    const int n = fftreg::kSizes[i];
    const int off = fftreg::tw_offset(n);
    for (int t = 0; t < n; ++t) {
      const double a = -2.0 * M_PI * double(t) / double(n);  // unit_roots, dft.hpp:39-47
      h[off + t] = make_float2(float(std::cos(a)), float(std::sin(a)));
    }
  }
  VXG_CUDA_CHECK(cudaMemcpyToSymbol(c_twiddle, h.data(), sizeof(float2) * h.size()));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
void encode_tensor_map_f32(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
                           const uint64_t* strides, const uint32_t* box) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    VXG_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc),
                                           cudaEnableDefault, &q));
    if (!enc) throw cuda_failure("cuTensorMapEncodeTiled unavailable");
  }
  cuuint64_t d[5], st[4];
  cuuint32_t bx[5], es[5];
  for (int k = 0; k < rank; ++k) {
    d[k] = dims[k];
    bx[k] = box[k];
    es[k] = 1;
    if (k < rank - 1) st[k] = strides[k];
  }
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, cuuint32_t(rank), const_cast<void*>(base), d, st,
                         bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw cuda_failure("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

namespace {

template <int T>
struct TileCfg {
  static constexpr int H = T / 2 + 1;                       // halved z extent
  static constexpr int SY = H | 1;                          // slot stride (odd)
  static constexpr int PADX = ((H - (T * SY) % 16) % 16 + 16) % 16;
  static constexpr int SX = T * SY + PADX;                  // x-plane stride
  static constexpr int NW = T * T * H;                      // frequencies per tile
  static constexpr int SMEM = T * SX * 8;                   // bytes
  static constexpr int THREADS = ((T * H + 31) / 32) * 32;  // one line per thread per pass
  static constexpr int MINB = T >= 28 ? 1 : (T >= 24 ? 2 : (T >= 20 ? 3 : 4));
  static __device__ __forceinline__ int idx(int kx, int ky, int kz) { return kx * SX + ky * SY + kz; }
};

// ---- K1 / K2: forward tile transform -----------------------------------------
template <int T>
__global__ void __launch_bounds__(TileCfg<T>::THREADS, TileCfg<T>::MINB)
    tile_fwd_kernel(FwdTileArgs a) {
  using C = TileCfg<T>;
  extern __shared__ float2 sp[];
  float* spf = reinterpret_cast<float*>(sp);
  const int64_t blk = blockIdx.x;
  const int64_t j = blk % a.f;
  const int64_t ml = blk / a.f;
  const int64_t m = a.m0 + ml;
  const int64_t s = m / a.tiles_per_img;
  const int64_t t = m % a.tiles_per_img;
  const int tz = int(t % a.ntz), ty = int((t / a.ntz) % a.nty), tx = int(t / (int64_t(a.ntz) * a.nty));
  const int ox = tx * a.vx, oy = ty * a.vy, oz = tz * a.vz;
  const float* img = a.src + (s * a.f + j) * a.img_stride;
  const int tid = threadIdx.x;

  // A0: real box -> slots (asynchronous 4-byte copies, zero outside the image).
  // Warp w owns x planes w, w + nwarps, ...; lane = z; rows advance by
  // pointer increments (no per-element index arithmetic).
  // (T > 32: the z rows take two lane passes)
  for (int zb = 0; zb < T; zb += 32) {
    constexpr int NWARPS = C::THREADS / 32;
    const int lane = (tid & 31) + zb, warp = tid >> 5;
    const int gz = oz + lane;
    if (ox + T <= a.nx && oy + T <= a.ny && oz + T <= a.nz) {
      // interior box (the common case): no bounds tests, one LDGSTS per row
      if (lane < T) {
        for (int x = warp; x < T; x += NWARPS) {
          const float* g = img + (int64_t(ox + x) * a.ny + oy) * a.pz + gz;
          float* d = spf + 2 * (x * C::SX) + lane;
#pragma unroll 8
          for (int y = 0; y < T; ++y) {
            cp_async4(d + 2 * C::SY * y, g, true);
            g += a.pz;
          }
        }
      }
    } else {
      const bool zin = lane < T && gz < a.nz;
      for (int x = warp; x < T; x += NWARPS) {
        const int gx = ox + x;
        const bool xin = zin && gx < a.nx;
        const float* g = img + (int64_t(gx) * a.ny + oy) * a.pz + gz;
        float* d = spf + 2 * (x * C::SX) + lane;
#pragma unroll 4
        for (int y = 0; y < T; ++y) {
          const bool in = xin && oy + y < a.ny;
          if (lane < T) cp_async4(d, in ? g : img, in);
          g += a.pz;
          d += 2 * C::SY;
        }
      }
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // A1: z r2c, lines l and l + T*T/2 share one complex transform (two-for-one)
  constexpr int LH = T * T / 2;
  if (tid < LH) {
    const int l1 = tid, l2 = tid + LH;
    float2* s1 = sp + (l1 / T) * C::SX + (l1 % T) * C::SY;
    float2* s2 = sp + (l2 / T) * C::SX + (l2 % T) * C::SY;
    float2 zz[T];
#pragma unroll
    for (int q = 0; q < T / 2; ++q) {
      const float2 r1 = s1[q], r2 = s2[q];
      zz[2 * q] = make_float2(r1.x, r2.x);
      zz[2 * q + 1] = make_float2(r1.y, r2.y);
    }
    fft<T, false>(zz);
#pragma unroll
    for (int k = 0; k < C::H; ++k) {
      const float2 zk = zz[k];
      const float2 zn = cconj(zz[(T - k) % T]);
      const float2 d = csub(zk, zn);
      s1[k] = make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y + zn.y));
      s2[k] = make_float2(0.5f * d.y, -0.5f * d.x);
    }
  }
  __syncthreads();

  // B: y lines (x, kz)
  if (tid < T * C::H) {
    const int kz = tid % C::H, x = tid / C::H;
    float2* base = sp + x * C::SX + kz;
    float2 v[T];
#pragma unroll
    for (int y = 0; y < T; ++y) v[y] = base[y * C::SY];
    fft<T, false>(v);
#pragma unroll
    for (int y = 0; y < T; ++y) base[y * C::SY] = v[y];
  }
  __syncthreads();

  // C: x lines (ky, kz), with the output scale
  if (tid < T * C::H) {
    const int kz = tid % C::H, ky = tid / C::H;
    float2* base = sp + ky * C::SY + kz;
    float2 v[T];
#pragma unroll
    for (int x = 0; x < T; ++x) v[x] = base[x * C::SX];
    fft<T, false>(v);
#pragma unroll
    for (int x = 0; x < T; ++x) base[x * C::SX] = make_float2(v[x].x * a.scale, v[x].y * a.scale);
  }
  __syncthreads();

  // D: spectrum chunks of lw frequencies (lw a power of two).  Thread t <
  // T*H owns (ky, kz) = (t / H, t % H) and walks kx: w = kx*T*H + t.
  const int lw = a.lw, lshift = __ffs(lw) - 1;
  float2* dst = a.out + (ml * a.f + j) * lw;
  const int64_t wb_stride = a.mstride * a.f * lw;
  if (tid < T * C::H) {
    const float2* s = sp + (tid / C::H) * C::SY + tid % C::H;
    if ((T * C::H) % 16 == 0 && lw == 16) {
      // kx steps move whole 16-frequency lines: a fixed pointer increment
      float2* o = dst + int64_t(tid >> 4) * wb_stride + (tid & 15);
      const int64_t step = int64_t((T * C::H) / 16) * wb_stride;
#pragma unroll 8
      for (int kx = 0; kx < T; ++kx) {
        *o = s[kx * C::SX];
        o += step;
      }
    } else {
      int w = tid;
#pragma unroll 4
      for (int kx = 0; kx < T; ++kx) {
        dst[int64_t(w >> lshift) * wb_stride + (w & (lw - 1))] = s[kx * C::SX];
        w += T * C::H;
      }
    }
  }
  // zero tail up to a multiple of lw (read by the FFMA contraction only)
  const int nwp = ((C::NW + lw - 1) / lw) * lw;
  if (tid < nwp - C::NW) {
    const int w = C::NW + tid;
    dst[int64_t(w >> lshift) * wb_stride + (w & (lw - 1))] = make_float2(0.f, 0.f);
  }
}

// ---- K1 / K2 on a CTA pair -------------------------------------------------------
// The same transform split over a 2-CTA cluster so that a tile's spectrum
// (139 KB at T = 32) becomes two 70 KB halves and two or three CTAs share an
// SM: their load / FFT / store phases then overlap, which one CTA per SM
// cannot do.  CTA rank r owns x-planes [r T/2, (r+1) T/2): it loads them, runs
// their z (two-for-one, lines y and y + T/2) and y passes, then after a
// cluster barrier transforms the x lines of its ky half, reading the other
// half of every line from the peer's shared memory (DSMEM), and stores the
// spectrum straight from registers.
template <int T>
struct PairCfg {
  using C = TileCfg<T>;
  static constexpr int HP = T / 2;                              // planes per CTA
  static constexpr int SMEM = HP * C::SX * 8;
  static constexpr int WORK = HP * C::H > HP * HP ? HP * C::H : HP * HP;
  // inverse with a pair-major spectrum: per kx one TMA box of the CTA's ky
  // half (HP*H complex), slabs padded to 128 bytes, staged in the plane buffer
  static constexpr int SL = ((HP * C::H * 8 + 127) / 128) * 128 / 8;
  static constexpr int SMEM_INV = (T * SL * 8 > SMEM ? T * SL * 8 : SMEM) + 16;
  static constexpr int THREADS = ((WORK + 31) / 32) * 32;
};

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t peer_addr(const void* local, unsigned peer) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local)), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(peer));
  return r;
}
__device__ __forceinline__ float2 ld_peer(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];\n" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}

template <int T>
__global__ void __launch_bounds__(PairCfg<T>::THREADS) tile_fwd_pair_kernel(FwdTileArgs a) {
  using C = TileCfg<T>;
  using P = PairCfg<T>;
  constexpr int HP = P::HP;
  constexpr int NWARPS = P::THREADS / 32;
  extern __shared__ float2 sp[];
  float* spf = reinterpret_cast<float*>(sp);
  const unsigned r = cluster_rank();
  const int64_t blk = blockIdx.x >> 1;
  const int64_t j = blk % a.f;
  const int64_t ml = blk / a.f;
  const int64_t m = a.m0 + ml;
  const int64_t s = m / a.tiles_per_img;
  const int64_t t = m % a.tiles_per_img;
  const int tz = int(t % a.ntz), ty = int((t / a.ntz) % a.nty), tx = int(t / (int64_t(a.ntz) * a.nty));
  const int ox = tx * a.vx + int(r) * HP, oy = ty * a.vy, oz = tz * a.vz;
  const float* img = a.src + (s * a.f + j) * a.img_stride;
  const int tid = threadIdx.x;

  // A0: this CTA's planes (raw) -> slots (T > 32: two lane passes per z row)
  for (int zb = 0; zb < T; zb += 32) {
    const int lane = (tid & 31) + zb, warp = tid >> 5;
    const int gz = oz + lane;
    if (ox + HP <= a.nx && oy + T <= a.ny && oz + T <= a.nz) {
      if (lane < T) {
        for (int x = warp; x < HP; x += NWARPS) {
          const float* g = img + (int64_t(ox + x) * a.ny + oy) * a.pz + gz;
          float* d = spf + 2 * (x * C::SX) + lane;
#pragma unroll 8
          for (int y = 0; y < T; ++y) {
            cp_async4(d + 2 * C::SY * y, g, true);
            g += a.pz;
          }
        }
      }
    } else {
      const bool zin = lane < T && gz < a.nz;
      for (int x = warp; x < HP; x += NWARPS) {
        const int gx = ox + x;
        const bool xin = zin && gx < a.nx;
        const float* g = img + (int64_t(gx) * a.ny + oy) * a.pz + gz;
        float* d = spf + 2 * (x * C::SX) + lane;
#pragma unroll 4
        for (int y = 0; y < T; ++y) {
          const bool in = xin && oy + y < a.ny;
          if (lane < T) cp_async4(d, in ? g : img, in);
          g += a.pz;
          d += 2 * C::SY;
        }
      }
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // A1: z r2c, lines (x, y) and (x, y + T/2) share one complex transform
  if (tid < HP * HP) {
    const int x = tid / HP, y = tid % HP;
    float2* s1 = sp + x * C::SX + y * C::SY;
    float2* s2 = s1 + HP * C::SY;
    float2 zz[T];
#pragma unroll
    for (int q = 0; q < T / 2; ++q) {
      const float2 r1 = s1[q], r2 = s2[q];
      zz[2 * q] = make_float2(r1.x, r2.x);
      zz[2 * q + 1] = make_float2(r1.y, r2.y);
    }
    fft<T, false>(zz);
#pragma unroll
    for (int k = 0; k < C::H; ++k) {
      const float2 zk = zz[k];
      const float2 zn = cconj(zz[(T - k) % T]);
      const float2 d = csub(zk, zn);
      s1[k] = make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y + zn.y));
      s2[k] = make_float2(0.5f * d.y, -0.5f * d.x);
    }
  }
  __syncthreads();

  // B: y lines (x, kz) of this CTA's planes
  if (tid < HP * C::H) {
    const int kz = tid % C::H, x = tid / C::H;
    float2* base = sp + x * C::SX + kz;
    float2 v[T];
#pragma unroll
    for (int y = 0; y < T; ++y) v[y] = base[y * C::SY];
    fft<T, false>(v);
#pragma unroll
    for (int y = 0; y < T; ++y) base[y * C::SY] = v[y];
  }
  // both halves transformed along z and y
  cluster_arrive();
  cluster_wait();

  // C: x lines (ky, kz) for ky in this CTA's half; x planes of the other half
  // come from the peer
  const int lw = a.lw, lshift = __ffs(lw) - 1;
  float2* dst = a.out + (ml * a.f + j) * lw;
  const int64_t wb_stride = a.mstride * a.f * lw;
  float2 v[T];
  const bool live = tid < HP * C::H;
  if (live) {
    const int ky = int(r) * HP + tid / C::H, kz = tid % C::H;
    const float2* base = sp + ky * C::SY + kz;
    const uint32_t pbase = peer_addr(base, r ^ 1u);
    if (r == 0) {
#pragma unroll
      for (int x = 0; x < HP; ++x) {
        v[x] = base[x * C::SX];
        v[HP + x] = ld_peer(pbase + uint32_t(x * C::SX * 8));
      }
    } else {
#pragma unroll
      for (int x = 0; x < HP; ++x) {
        v[x] = ld_peer(pbase + uint32_t(x * C::SX * 8));
        v[HP + x] = base[x * C::SX];
      }
    }
  }
  cluster_arrive();  // my reads of the peer are issued; it may exit after its own wait
  if (live) {
    fft<T, false>(v);
    const int t0 = int(r) * HP * C::H + tid;  // w = kx*T*H + t0
    if ((T * C::H) % 16 == 0 && lw == 16) {
      float2* o = dst + int64_t(t0 >> 4) * wb_stride + (t0 & 15);
      const int64_t step = int64_t((T * C::H) / 16) * wb_stride;
#pragma unroll
      for (int kx = 0; kx < T; ++kx) {
        *o = make_float2(v[kx].x * a.scale, v[kx].y * a.scale);
        o += step;
      }
    } else {
      int w = t0;
#pragma unroll
      for (int kx = 0; kx < T; ++kx) {
        dst[int64_t(w >> lshift) * wb_stride + (w & (lw - 1))] = make_float2(v[kx].x * a.scale, v[kx].y * a.scale);
        w += T * C::H;
      }
    }
  }
  if (r == 0) {
    const int nwp = ((C::NW + lw - 1) / lw) * lw;
    if (tid < nwp - C::NW) {
      const int w = C::NW + tid;
      dst[int64_t(w >> lshift) * wb_stride + (w & (lw - 1))] = make_float2(0.f, 0.f);
    }
  }
  cluster_wait();  // the peer finished reading my planes
}

// ---- K4: inverse tile transform with crop + bias + ReLU ------------------------
template <int T>
__global__ void __launch_bounds__(TileCfg<T>::THREADS, TileCfg<T>::MINB)
    tile_inv_kernel(InvTileArgs a) {
  using C = TileCfg<T>;
  extern __shared__ float2 sp[];
  float* spf = reinterpret_cast<float*>(sp);
  const int64_t blk = blockIdx.x;
  const int64_t i = blk % a.fo;
  const int64_t ml = blk / a.fo;
  const int64_t m = a.m0 + ml;
  const int64_t s = m / a.tiles_per_img;
  const int64_t t = m % a.tiles_per_img;
  const int tz = int(t % a.ntz), ty = int((t / a.ntz) % a.nty), tx = int(t / (int64_t(a.ntz) * a.nty));
  const int tid = threadIdx.x;

  // A: spectrum lines -> smem (asynchronous 8-byte copies); with a single
  // input map (a.wsp) or direct_x the x pass loads from HBM itself instead
  const int lw = a.lw, lshift = __ffs(lw) - 1;
  const float2* src = a.spec + (ml * a.fo + i) * lw;
  const int64_t wb_stride = a.mstride * a.fo * lw;
  if (tid < T * C::H && !a.wsp && !a.direct_x) {
    float2* s = sp + (tid / C::H) * C::SY + tid % C::H;
    if ((T * C::H) % 16 == 0 && lw == 16) {
      const float2* g = src + int64_t(tid >> 4) * wb_stride + (tid & 15);
      const int64_t step = int64_t((T * C::H) / 16) * wb_stride;
#pragma unroll 8
      for (int kx = 0; kx < T; ++kx) {
        cp_async8(s + kx * C::SX, g);
        g += step;
      }
    } else {
      int w = tid;
#pragma unroll 4
      for (int kx = 0; kx < T; ++kx) {
        cp_async8(s + kx * C::SX, src + int64_t(w >> lshift) * wb_stride + (w & (lw - 1)));
        w += T * C::H;
      }
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // B: x lines, all (ky, kz)
  if (tid < T * C::H) {
    const int kz = tid % C::H, ky = tid / C::H;
    float2* base = sp + ky * C::SY + kz;
    float2 v[T];
    if (a.wsp) {
      // f = 1: Y[w](row, i) = X[w](row) W[w](i) (lw = 16), w = kx*T*H + tid
      const float2* sx = a.spec + ml * 16;
      const float2* sw = a.wsp + i * 16;
      const int64_t xs = a.mstride * 16, ws = a.w_fo * 16;
#pragma unroll
      for (int x = 0; x < T; ++x) {
        const int w = x * T * C::H + tid;
        v[x] = cmul(__ldg(sx + int64_t(w >> 4) * xs + (w & 15)), __ldg(sw + int64_t(w >> 4) * ws + (w & 15)));
      }
    } else if (a.direct_x) {
      // straight from HBM into registers: no shared-memory round trip
      int w = tid;
#pragma unroll
      for (int x = 0; x < T; ++x) {
        v[x] = __ldg(src + int64_t(w >> lshift) * wb_stride + (w & (lw - 1)));
        w += T * C::H;
      }
    } else {
#pragma unroll
      for (int x = 0; x < T; ++x) v[x] = base[x * C::SX];
    }
    fft<T, true>(v);
#pragma unroll
    for (int x = 0; x < T; ++x) base[x * C::SX] = v[x];
  }
  __syncthreads();

  // C: y lines only for x inside the crop
  if (tid < a.vx * C::H) {
    const int kz = tid % C::H, x = a.cx + tid / C::H;
    float2* base = sp + x * C::SX + kz;
    float2 v[T];
#pragma unroll
    for (int y = 0; y < T; ++y) v[y] = base[y * C::SY];
    fft<T, true>(v);
#pragma unroll
    for (int y = 0; y < T; ++y) base[y * C::SY] = v[y];
  }
  __syncthreads();

  // D: z c2r for (x, y) inside the crop, pairs (l, l + half); bias + activation
  const int L = a.vx * a.vy;
  const int half = (L + 1) / 2;
  if (tid < half) {
    const float bias = __ldg(a.bias + i);
    const int l1 = tid, l2 = tid + half;
    const bool has2 = l2 < L;
    float2* s1 = sp + (a.cx + l1 / a.vy) * C::SX + (a.cy + l1 % a.vy) * C::SY;
    float2* s2 = has2 ? sp + (a.cx + l2 / a.vy) * C::SX + (a.cy + l2 % a.vy) * C::SY : s1;
    float2 zz[T];
#pragma unroll
    for (int k = 0; k < C::H; ++k) {
      const float2 A = s1[k];
      const float2 B = has2 ? s2[k] : make_float2(0.f, 0.f);
      zz[k] = make_float2(A.x - B.y, A.y + B.x);  // A + iB
    }
#pragma unroll
    for (int k = C::H; k < T; ++k) {
      const float2 A = s1[T - k];
      const float2 B = has2 ? s2[T - k] : make_float2(0.f, 0.f);
      zz[k] = make_float2(A.x + B.y, -A.y + B.x);  // conj(A) + i conj(B)
    }
    fft<T, true>(zz);
    float* r1 = spf + 2 * (s1 - sp);
    float* r2 = spf + 2 * (s2 - sp);
#pragma unroll
    for (int z = 0; z < T; ++z) {
      if (z >= a.cz && z < a.cz + a.vz) {
        const float v1 = zz[z].x + bias;
        r1[z] = a.relu ? (v1 > 0.f ? v1 : 0.f) : v1;  // activate (layers.hpp:105-108)
        if (has2) {
          const float v2 = zz[z].y + bias;
          r2[z] = a.relu ? (v2 > 0.f ? v2 : 0.f) : v2;
        }
      }
    }
  }
  __syncthreads();

  // E: store of the crop, clipped to the output image: warp w owns x planes
  // w, w + nwarps, ...; lane = z; rows advance by pointer increments.
  // (T > 32: the z rows take two lane passes)
  for (int zb = 0; zb < T; zb += 32) {
    constexpr int NWARPS = C::THREADS / 32;
    const int lane = (tid & 31) + zb, warp = tid >> 5;
    const int gx0 = tx * a.vx, gy0 = ty * a.vy, gz = tz * a.vz + lane;
    const bool zin = lane < a.vz && gz < a.onz;
    const int ylim = min(a.vy, a.ony - gy0);
    for (int x = warp; x < a.vx; x += NWARPS) {
      const int gx = gx0 + x;
      if (!zin || gx >= a.onx) continue;
      float* o = a.dst + (s * a.fo + i) * a.oel + (int64_t(gx) * a.ony + gy0) * a.opz + gz;
      const float* r = spf + 2 * ((a.cx + x) * C::SX + a.cy * C::SY) + a.cz + lane;
#pragma unroll 4
      for (int y = 0; y < ylim; ++y) {
        *o = *r;
        o += a.opz;
        r += 2 * C::SY;
      }
    }
  }
}

// ---- K4 on a CTA pair ---------------------------------------------------------
// Rank r transforms the x lines of its ky half straight from HBM into registers
// (one coalesced 8-byte load per line element, 32 in flight per thread),
// writes each result to the CTA owning its x plane (local or DSMEM), and after
// a cluster barrier runs the y pass, the z c2r with bias + activation and the
// store for the crop planes it owns.
__device__ __forceinline__ void st_peer(uint32_t addr, float2 v) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};\n" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}

template <int T>
__global__ void __launch_bounds__(PairCfg<T>::THREADS) tile_inv_pair_kernel(InvTileArgs a,
                                                                           const __grid_constant__ CUtensorMap ymap) {
  using C = TileCfg<T>;
  using P = PairCfg<T>;
  constexpr int HP = P::HP;
  constexpr int NWARPS = P::THREADS / 32;
  extern __shared__ float2 sp[];
  float* spf = reinterpret_cast<float*>(sp);
  const unsigned r = cluster_rank();
  const int64_t blk = blockIdx.x >> 1;
  const int64_t i = blk % a.fo;
  const int64_t ml = blk / a.fo;
  const int64_t m = a.m0 + ml;
  const int64_t s = m / a.tiles_per_img;
  const int64_t t = m % a.tiles_per_img;
  const int tz = int(t % a.ntz), ty = int((t / a.ntz) % a.nty), tx = int(t / (int64_t(a.ntz) * a.nty));
  const int tid = threadIdx.x;
  const int x0 = int(r) * HP;  // my planes [x0, x0 + HP)

  // A+B: x lines (ky in my half, all kz) from HBM, inverse transform, scatter
  float2 v[T];
  const bool tma = a.lw == 2;
  if (tma) {
    // pair-major spectrum: the copy engine gathers the 16-byte pieces of my
    // x lines (one box per kx) into the plane buffer, used as staging
    uint64_t& bar = *reinterpret_cast<uint64_t*>(spf + 2 * ((P::SMEM_INV - 16) / 8));
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(T * HP * C::H * 8));
      for (int kx = 0; kx < T; ++kx) {
        const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sp + kx * P::SL));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(d),
            "l"(&ymap), "r"(0), "r"(int(i)), "r"(int(ml)), "r"((kx * T * C::H + x0 * C::H) / 2), "r"(b)
            : "memory");
      }
    }
    __syncthreads();
    asm volatile(
        "{\n\t.reg .pred P;\nWTI_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra WTI_%=;\n\t}\n" ::"r"(b)
        : "memory");
    if (tid < HP * C::H) {
#pragma unroll
      for (int kx = 0; kx < T; ++kx) v[kx] = sp[kx * P::SL + tid];
    }
    // both CTAs have read their staging before either scatters into the other
    cluster_arrive();
    cluster_wait();
  }
  if (tid < HP * C::H) {
    const int lw = a.lw, lshift = __ffs(lw) - 1;
    const float2* src = a.spec + (ml * a.fo + i) * lw;
    const int64_t wb_stride = a.mstride * a.fo * lw;
    const int t0 = x0 * C::H + tid;  // ky * H + kz, ky = x0 + tid / H
    if (a.wsp) {
      // f = 1: Y[w](row, i) = X[w](row) W[w](i), formed on load (lw = 16)
      const float2* sx = a.spec + ml * 16;
      const float2* sw = a.wsp + i * 16;
      const int64_t xs = a.mstride * 16, ws = a.w_fo * 16;
#pragma unroll
      for (int kx = 0; kx < T; ++kx) {
        const int w = kx * T * C::H + t0;
        v[kx] = cmul(__ldg(sx + int64_t(w >> 4) * xs + (w & 15)), __ldg(sw + int64_t(w >> 4) * ws + (w & 15)));
      }
    } else if (tma) {
    } else if ((T * C::H) % 16 == 0 && lw == 16) {
      const float2* g = src + int64_t(t0 >> 4) * wb_stride + (t0 & 15);
      const int64_t step = int64_t((T * C::H) / 16) * wb_stride;
#pragma unroll
      for (int kx = 0; kx < T; ++kx) v[kx] = __ldg(g + kx * step);
    } else {
#pragma unroll
      for (int kx = 0; kx < T; ++kx) {
        const int w = kx * T * C::H + t0;
        v[kx] = __ldg(src + int64_t(w >> lshift) * wb_stride + (w & (lw - 1)));
      }
    }
    fft<T, true>(v);
    const int ky = x0 + tid / C::H, kz = tid % C::H;
    float2* base = sp + ky * C::SY + kz;
    const uint32_t pbase = peer_addr(base, r ^ 1u);
    if (r == 0) {
#pragma unroll
      for (int x = 0; x < HP; ++x) {
        base[x * C::SX] = v[x];
        st_peer(pbase + uint32_t(x * C::SX * 8), v[HP + x]);
      }
    } else {
#pragma unroll
      for (int x = 0; x < HP; ++x) {
        st_peer(pbase + uint32_t(x * C::SX * 8), v[x]);
        base[x * C::SX] = v[HP + x];
      }
    }
  }
  cluster_arrive();
  cluster_wait();

  // crop planes owned here
  const int xa = max(a.cx, x0), xb = min(a.cx + a.vx, x0 + HP);
  const int nxl = max(0, xb - xa);

  // C: y lines for my crop planes
  if (tid < nxl * C::H) {
    const int kz = tid % C::H, xl = xa - x0 + tid / C::H;
    float2* base = sp + xl * C::SX + kz;
    float2 v[T];
#pragma unroll
    for (int y = 0; y < T; ++y) v[y] = base[y * C::SY];
    fft<T, true>(v);
#pragma unroll
    for (int y = 0; y < T; ++y) base[y * C::SY] = v[y];
  }
  __syncthreads();

  // D: z c2r for crop (x, y) of my planes, pairs (l, l + half); bias + activation
  const int L = nxl * a.vy;
  const int half = (L + 1) / 2;
  for (int l1 = tid; l1 < half; l1 += P::THREADS) {
    const float bias = __ldg(a.bias + i);
    const int l2 = l1 + half;
    const bool has2 = l2 < L;
    float2* s1 = sp + (xa - x0 + l1 / a.vy) * C::SX + (a.cy + l1 % a.vy) * C::SY;
    float2* s2 = has2 ? sp + (xa - x0 + l2 / a.vy) * C::SX + (a.cy + l2 % a.vy) * C::SY : s1;
    float2 zz[T];
#pragma unroll
    for (int k = 0; k < C::H; ++k) {
      const float2 A = s1[k];
      const float2 B = has2 ? s2[k] : make_float2(0.f, 0.f);
      zz[k] = make_float2(A.x - B.y, A.y + B.x);  // A + iB
    }
#pragma unroll
    for (int k = C::H; k < T; ++k) {
      const float2 A = s1[T - k];
      const float2 B = has2 ? s2[T - k] : make_float2(0.f, 0.f);
      zz[k] = make_float2(A.x + B.y, -A.y + B.x);  // conj(A) + i conj(B)
    }
    fft<T, true>(zz);
    float* r1 = spf + 2 * (s1 - sp);
    float* r2 = spf + 2 * (s2 - sp);
#pragma unroll
    for (int z = 0; z < T; ++z) {
      if (z >= a.cz && z < a.cz + a.vz) {
        const float v1 = zz[z].x + bias;
        r1[z] = a.relu ? (v1 > 0.f ? v1 : 0.f) : v1;  // activate (layers.hpp:105-108)
        if (has2) {
          const float v2 = zz[z].y + bias;
          r2[z] = a.relu ? (v2 > 0.f ? v2 : 0.f) : v2;
        }
      }
    }
  }
  __syncthreads();

  // E: store my crop planes, clipped to the output image (vz > 32: two lane passes)
  for (int zb = 0; zb < T; zb += 32) {
    const int lane = (tid & 31) + zb, warp = tid >> 5;
    const int gy0 = ty * a.vy, gz = tz * a.vz + lane;
    const bool zin = lane < a.vz && gz < a.onz;
    const int ylim = min(a.vy, a.ony - gy0);
    for (int xx = warp; xx < nxl; xx += NWARPS) {
      const int gx = tx * a.vx + (xa - a.cx) + xx;
      if (!zin || gx >= a.onx) continue;
      float* o = a.dst + (s * a.fo + i) * a.oel + (int64_t(gx) * a.ony + gy0) * a.opz + gz;
      const float* rr = spf + 2 * ((xa - x0 + xx) * C::SX + a.cy * C::SY) + a.cz + lane;
#pragma unroll 4
      for (int y = 0; y < ylim; ++y) {
        *o = *rr;
        o += a.opz;
        rr += 2 * C::SY;
      }
    }
  }
}

// T whose whole spectrum fits one CTA's shared memory (else: CTA pairs only)
template <int T>
constexpr bool single_fits() {
  return TileCfg<T>::SMEM <= 232448 && TileCfg<T>::THREADS <= 1024;
}

template <int T>
void fwd_t(Ctx* c, const FwdTileArgs& a, int64_t nblocks) {
  using C = TileCfg<T>;
  if ((a.pair && T >= 24) || !single_fits<T>()) {
    using P = PairCfg<T>;
    static PerDeviceOnce pconf;
    if (pconf.first()) {
      VXG_CUDA_CHECK(cudaFuncSetAttribute(tile_fwd_pair_kernel<T>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM));
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(2 * nblocks));
    cfg.blockDim = dim3(P::THREADS);
    cfg.dynamicSmemBytes = P::SMEM;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    VXG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, tile_fwd_pair_kernel<T>, a));
    c->counted();
    check_launch("tile_fwd_pair_kernel");
    return;
  }
  if constexpr (single_fits<T>()) {
    static PerDeviceOnce configured;
    if (configured.first()) {
      VXG_CUDA_CHECK(cudaFuncSetAttribute(tile_fwd_kernel<T>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    }
    tile_fwd_kernel<T><<<unsigned(nblocks), C::THREADS, C::SMEM, c->stream>>>(a);
    c->counted();
    check_launch("tile_fwd_kernel");
  }
}

template <int T>
void inv_t(Ctx* c, const InvTileArgs& a, int64_t nblocks) {
  using C = TileCfg<T>;
  if ((a.pair && T >= 24) || !single_fits<T>()) {
    using P = PairCfg<T>;
    static PerDeviceOnce pconf;
    if (pconf.first()) {
      VXG_CUDA_CHECK(cudaFuncSetAttribute(tile_inv_pair_kernel<T>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, P::SMEM_INV));
    }
    CUtensorMap ymap{};
    if (a.lw == 2) {
      // pair-major Y: {4 floats of a pair, fo maps, mstride rows, pairs}
      const uint64_t dims[4] = {4, uint64_t(a.fo), uint64_t(a.mstride), uint64_t(a.nwp) / 2};
      const uint64_t strides[3] = {16, uint64_t(a.fo) * 16, uint64_t(a.mstride) * a.fo * 16};
      const uint32_t box[4] = {4, 1, 1, uint32_t(P::HP * TileCfg<T>::H / 2)};
      encode_tensor_map_f32(&ymap, a.spec, 4, dims, strides, box);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(2 * nblocks));
    cfg.blockDim = dim3(P::THREADS);
    cfg.dynamicSmemBytes = P::SMEM_INV;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    VXG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, tile_inv_pair_kernel<T>, a, ymap));
    c->counted();
    check_launch("tile_inv_pair_kernel");
    return;
  }
  if constexpr (single_fits<T>()) {
    static PerDeviceOnce configured;
    if (configured.first()) {
      VXG_CUDA_CHECK(cudaFuncSetAttribute(tile_inv_kernel<T>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    }
    tile_inv_kernel<T><<<unsigned(nblocks), C::THREADS, C::SMEM, c->stream>>>(a);
    c->counted();
    check_launch("tile_inv_kernel");
  }
}

}  // namespace

bool tile_pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VXG_TILE_PAIR");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return on;
}

bool inv_pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VXG_INV_PAIR");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return on;
}

// supported tile FFT sizes (even, {2,3,5,7}-smooth)
// 36 and 40 run on CTA pairs only (a whole 40^3 spectrum exceeds one CTA's
// shared memory): the big-kernel nets (k = 7, 9) waste less overlap-save work
const int kTileSizes[] = {4, 6, 8, 10, 12, 16, 20, 24, 28, 30, 32, 36, 40};
const int kNumTileSizes = sizeof(kTileSizes) / sizeof(int);

int64_t tile_nwp(int T, int lw) {
  const int64_t nw = int64_t(T) * T * (T / 2 + 1);
  return ((nw + lw - 1) / lw) * lw;
}

#define VXG_TILE_SWITCH(FN)                                         \
  switch (T) {                                                      \
    case 4: FN<4>(c, a, nblocks); break;                            \
    case 6: FN<6>(c, a, nblocks); break;                            \
    case 8: FN<8>(c, a, nblocks); break;                            \
    case 10: FN<10>(c, a, nblocks); break;                          \
    case 12: FN<12>(c, a, nblocks); break;                          \
    case 16: FN<16>(c, a, nblocks); break;                          \
    case 20: FN<20>(c, a, nblocks); break;                          \
    case 24: FN<24>(c, a, nblocks); break;                          \
    case 28: FN<28>(c, a, nblocks); break;                          \
    case 30: FN<30>(c, a, nblocks); break;                          \
    case 32: FN<32>(c, a, nblocks); break;                          \
    case 36: FN<36>(c, a, nblocks); break;                          \
    case 40: FN<40>(c, a, nblocks); break;                          \
    default: throw invalid("tile fft: unsupported tile size");      \
  }

void launch_tile_fwd(Ctx* c, int T, const FwdTileArgs& a, int64_t nblocks) {
  const double nw = double(T) * T * (T / 2 + 1);
  KScope ks(c, a.kind, 0.0, double(nblocks) * (4.0 * double(T) * T * T + 8.0 * nw));
  VXG_TILE_SWITCH(fwd_t)
}

void launch_tile_inv(Ctx* c, int T, const InvTileArgs& a0, int64_t nblocks) {
  // The one-CTA inverse loads its x lines from HBM straight into registers at
  // T >= 28 (T = 30 / 36: -7 / -9 % inverse time) and stages them through
  // shared memory below (T = 16: +4 % direct), profiles/r2_experiments.md §17;
  // VXG_INV_DIRECT=0/1 forces either
  InvTileArgs a = a0;
  {
    const char* e = std::getenv("VXG_INV_DIRECT");
    a.direct_x = e ? std::strcmp(e, "1") == 0 : T >= 28;
  }
  const double nw = double(T) * T * (T / 2 + 1);
  KScope ks(c, VXG_K_TILE_INV, 0.0,
            double(nblocks) * (8.0 * nw + 4.0 * double(a.vx) * a.vy * a.vz));
  VXG_TILE_SWITCH(inv_t)
}

}  // namespace vxg
