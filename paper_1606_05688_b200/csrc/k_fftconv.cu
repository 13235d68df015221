// K1-K4: tiled pruned-FFT convolution.
//
// Math of conv_fft_data_parallel / conv_fft_staged / conv_fft_task_parallel
// (proj/include/voxin/layers.hpp:203-371, task_conv.hpp:415-442): valid
// convolution = crop of the circular convolution of zero-padded spectra.  The
// reference pads the WHOLE image to N(n) and multi-passes every axis through
// memory; here the output is cut into overlap-save tiles of a cubic FFT size
// T (T - k + 1 valid outputs per axis per tile), so that
//   * each 3D transform runs entirely on-chip (one HBM read of the tile, one
//     write of its spectrum) -- K1 tile_fwd_kernel, K4 tile_inv_kernel;
//   * kernel spectra are small (T^3) and computed once per layer (K2 = the
//     same forward kernel on the k^3 kernels, pruned by zero fill), scaled by
//     1/T^3 so the inverse needs no extra pass;
//   * the per-frequency multiply-accumulate becomes, for every frequency w, a
//     real GEMM-shaped complex contraction Y[w](m, i) = sum_j X[w](m, j) W[w](i, j)
//     over M = S * tiles rows -- K3 cgemm_kernel (fp32 FFMA).
// Spectra live in HBM as [w/16][m][channel][w%16] complex64 so every producer
// and consumer moves whole 128-byte lines.  The inverse keeps only the valid
// region (pruned lines) and fuses crop + bias + ReLU into its store
// (layers.hpp:256-260, 355-361).
#include <cmath>
#include <vector>

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
      const double a = -2.0 * M_PI * double(t) / double(n);
      h[off + t] = make_float2(float(std::cos(a)), float(std::sin(a)));
    }
  }
  VXG_CUDA_CHECK(cudaMemcpyToSymbol(c_twiddle, h.data(), sizeof(float2) * h.size()));
}

namespace {

constexpr int WB = 16;  // frequencies per 128-byte spectrum line

template <int T>
struct TileCfg {
  static constexpr int H = T / 2 + 1;                      // halved z extent
  static constexpr int SY = H;                             // smem stride of y (complex)
  static constexpr int PADX = ((H - (T * H) % 16) % 16 + 16) % 16;
  static constexpr int SX = T * H + PADX;                  // smem stride of x (complex)
  static constexpr int NW = T * T * H;                     // frequencies per tile
  static constexpr int NWB = (NW + WB - 1) / WB;
  static constexpr int SMEM = T * SX * 8;                  // bytes
};

constexpr int kFftThreads = 256;

// cp.async (LDGSTS) helpers: asynchronous global -> shared copies that need no
// registers, so a thread can keep dozens of loads in flight.  pred == false
// zero-fills the destination (src-size 0).
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = pred ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// two CTAs per SM whenever the spectrum fits in half the shared memory
template <int T>
constexpr int fft_min_blocks() { return T <= 28 ? 2 : 1; }

// ---- K1 / K2: forward tile transform -----------------------------------------
//
// One CTA per (tile m, channel j).  A0 stages the real T^3 box (zero outside
// the image) with coalesced loads, each z line inside its own complex slot;
// A1 transforms pairs of real z lines with one complex FFT (two-for-one r2c);
// B / C run the y and x lines in shared memory; D stores the spectrum lines.
template <int T>
__global__ void __launch_bounds__(kFftThreads, fft_min_blocks<T>()) tile_fwd_kernel(FwdTileArgs a) {
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

  // A0: real box -> slots, asynchronous 4-byte copies (zero-filled outside
  // the image) so every thread keeps all of its loads in flight at once
#pragma unroll 8
  for (int idx = threadIdx.x; idx < T * T * T; idx += kFftThreads) {
    const int z = idx % T, l = idx / T;
    const int y = l % T, x = l / T;
    const int gx = ox + x, gy = oy + y, gz = oz + z;
    const bool in = gx < a.nx && gy < a.ny && gz < a.nz;
    const float* g = in ? img + (int64_t(gx) * a.ny + gy) * a.nz + gz : img;
    cp_async4(spf + 2 * (x * C::SX + y * C::SY) + z, g, in);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // A1: z r2c, lines l and l + T*T/2 share one complex transform
  constexpr int LH = T * T / 2;
  for (int p = threadIdx.x; p < LH; p += kFftThreads) {
    const int l1 = p, l2 = p + LH;
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

  // B: y lines for every (x, kz)
  for (int l = threadIdx.x; l < T * C::H; l += kFftThreads) {
    const int kz = l % C::H, x = l / C::H;
    float2* base = sp + x * C::SX + kz;
    float2 v[T];
#pragma unroll
    for (int y = 0; y < T; ++y) v[y] = base[y * C::SY];
    fft<T, false>(v);
#pragma unroll
    for (int y = 0; y < T; ++y) base[y * C::SY] = v[y];
  }
  __syncthreads();

  // C: x lines for every (ky, kz), with the output scale
  for (int l = threadIdx.x; l < T * C::H; l += kFftThreads) {
    float2* base = sp + l;  // ky * SY + kz == l
    float2 v[T];
#pragma unroll
    for (int x = 0; x < T; ++x) v[x] = base[x * C::SX];
    fft<T, false>(v);
#pragma unroll
    for (int x = 0; x < T; ++x) base[x * C::SX] = make_float2(v[x].x * a.scale, v[x].y * a.scale);
  }
  __syncthreads();

  // D: spectrum lines, w = (kx*T + ky)*H + kz, zero tail up to NWB*16
  float2* dst = a.out + (ml * a.f + j) * WB;
  const int64_t wb_stride = a.mstride * a.f * WB;
  for (int w = threadIdx.x; w < C::NWB * WB; w += kFftThreads) {
    float2 v = make_float2(0.f, 0.f);
    if (w < C::NW) v = sp[(w / (T * C::H)) * C::SX + w % (T * C::H)];
    dst[(w / WB) * wb_stride + (w % WB)] = v;
  }
}

// ---- K4: inverse tile transform with crop + bias + ReLU ------------------------
//
// A loads the product spectrum of (tile m, output map i); B inverts every x
// line; C inverts y lines only for x inside the valid crop; D inverts pairs of
// z lines (two-for-one c2r) only for (x, y) inside the crop and applies
// bias + activation; E stores the crop coalesced and clipped to the image.
template <int T>
__global__ void __launch_bounds__(kFftThreads, fft_min_blocks<T>()) tile_inv_kernel(InvTileArgs a) {
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

  // A: spectrum lines -> smem, asynchronous 8-byte copies
  const float2* src = a.spec + (ml * a.fo + i) * WB;
  const int64_t wb_stride = a.mstride * a.fo * WB;
#pragma unroll 8
  for (int w = threadIdx.x; w < C::NW; w += kFftThreads)
    cp_async8(sp + (w / (T * C::H)) * C::SX + w % (T * C::H), src + (w / WB) * wb_stride + (w % WB));
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // B: x lines, all (ky, kz)
  for (int l = threadIdx.x; l < T * C::H; l += kFftThreads) {
    float2* base = sp + l;
    float2 v[T];
#pragma unroll
    for (int x = 0; x < T; ++x) v[x] = base[x * C::SX];
    fft<T, true>(v);
#pragma unroll
    for (int x = 0; x < T; ++x) base[x * C::SX] = v[x];
  }
  __syncthreads();

  // C: y lines for x in the crop
  for (int l = threadIdx.x; l < a.vx * C::H; l += kFftThreads) {
    const int kz = l % C::H, x = a.cx + l / C::H;
    float2* base = sp + x * C::SX + kz;
    float2 v[T];
#pragma unroll
    for (int y = 0; y < T; ++y) v[y] = base[y * C::SY];
    fft<T, true>(v);
#pragma unroll
    for (int y = 0; y < T; ++y) base[y * C::SY] = v[y];
  }
  __syncthreads();

  // D: z c2r for (x, y) in the crop, pairs (l, l + half)
  const int L = a.vx * a.vy;
  const int half = (L + 1) / 2;
  const float bias = __ldg(a.bias + i);
  for (int p = threadIdx.x; p < half; p += kFftThreads) {
    const int l1 = p, l2 = p + half;
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
        r1[z] = a.relu ? (v1 > 0.f ? v1 : 0.f) : v1;
      }
    }
    if (has2) {
#pragma unroll
      for (int z = 0; z < T; ++z) {
        if (z >= a.cz && z < a.cz + a.vz) {
          const float v2 = zz[z].y + bias;
          r2[z] = a.relu ? (v2 > 0.f ? v2 : 0.f) : v2;
        }
      }
    }
  }
  __syncthreads();

  // E: coalesced store of the crop, clipped to the output image
  float* out = a.dst + (s * a.fo + i) * a.oel;
  const int gx0 = tx * a.vx, gy0 = ty * a.vy, gz0 = tz * a.vz;
  const int V = a.vx * a.vy * a.vz;
  for (int idx = threadIdx.x; idx < V; idx += kFftThreads) {
    const int z = idx % a.vz, l = idx / a.vz;
    const int y = l % a.vy, x = l / a.vy;
    const int gx = gx0 + x, gy = gy0 + y, gz = gz0 + z;
    if (gx < a.onx && gy < a.ony && gz < a.onz)
      out[(int64_t(gx) * a.ony + gy) * a.onz + gz] =
          spf[2 * ((a.cx + x) * C::SX + (a.cy + y) * C::SY) + a.cz + z];
  }
}

// ---- K3: per-frequency complex contraction (fp32 FFMA) -------------------------
//
// CTA = 16 frequencies (one 128-byte spectrum line) x MB rows x IB output maps,
// all f input maps in JC-deep stages double-buffered with cp.async.  Thread =
// one frequency x MT rows x IT maps (MT*IT complex accumulators, 4 FFMA per
// complex MAC).  Grid order keeps all m-blocks of one frequency block adjacent
// so the kernel-spectrum block stays L2-resident while X streams from HBM.

template <int MT, int IT, int MB, int IB, int JC>
struct GemmCfg {
  static constexpr int THREADS = WB * (MB / MT) * (IB / IT);
  static constexpr int XS = JC * MB * WB;  // complex per stage
  static constexpr int WS = JC * IB * WB;
  static constexpr int SMEM = 2 * (XS + WS) * 8;
};

template <int MT, int IT, int MB, int IB, int JC>
__global__ void __launch_bounds__(GemmCfg<MT, IT, MB, IB, JC>::THREADS)
    cgemm_kernel(GemmArgs a) {
  using G = GemmCfg<MT, IT, MB, IB, JC>;
  extern __shared__ float2 sm[];
  float2* xs = sm;                  // [2][JC][MB][WB]
  float2* ws = sm + 2 * G::XS;      // [2][JC][IB][WB]

  const int64_t bx = blockIdx.x;
  const int64_t mb = bx % a.mblocks;
  const int64_t ib = (bx / a.mblocks) % a.iblocks;
  const int64_t wb = bx / (int64_t(a.mblocks) * a.iblocks);
  const int64_t m0 = mb * MB;
  const int i0 = int(ib * IB);

  const int tid = threadIdx.x;
  const int w = tid % WB;
  const int sub = tid / WB;
  const int mi = sub % (MB / MT);
  const int ii = sub / (MB / MT);

  const float2* X = a.X + wb * a.mstride * a.f * WB;
  const float2* W = a.W + wb * int64_t(a.fo) * a.f * WB;

  auto load_stage = [&](int stage, int j0) {
    float2* xd = xs + stage * G::XS;
    float2* wd = ws + stage * G::WS;
    // X rows: (jj, mm) -> 8 chunks of 16 B
    for (int c = tid; c < JC * MB * 8; c += G::THREADS) {
      const int part = c % 8, row = c / 8;
      const int mm = row % MB, jj = row / MB;
      const int64_t m = m0 + mm;
      const int j = j0 + jj;
      const bool ok = m < a.M && j < a.f;
      const float2* g = ok ? X + (m * a.f + j) * WB + part * 2 : a.X;
      cp_async16(xd + (jj * MB + mm) * WB + part * 2, g, ok);
    }
    for (int c = tid; c < JC * IB * 8; c += G::THREADS) {
      const int part = c % 8, row = c / 8;
      const int i2 = row % IB, jj = row / IB;
      const int i = i0 + i2;
      const int j = j0 + jj;
      const bool ok = i < a.fo && j < a.f;
      const float2* g = ok ? W + (int64_t(i) * a.f + j) * WB + part * 2 : a.W;
      cp_async16(wd + (jj * IB + i2) * WB + part * 2, g, ok);
    }
    cp_async_commit();
  };

  float2 acc[MT][IT];
#pragma unroll
  for (int r = 0; r < MT; ++r)
#pragma unroll
    for (int c = 0; c < IT; ++c) acc[r][c] = make_float2(0.f, 0.f);

  const int nstages = (a.f + JC - 1) / JC;
  load_stage(0, 0);
  for (int st = 0; st < nstages; ++st) {
    const int cur = st & 1;
    if (st + 1 < nstages) {
      load_stage(cur ^ 1, (st + 1) * JC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float2* xd = xs + cur * G::XS;
    const float2* wd = ws + cur * G::WS;
#pragma unroll 2
    for (int jj = 0; jj < JC; ++jj) {
      float2 xa[MT], wa[IT];
#pragma unroll
      for (int r = 0; r < MT; ++r) xa[r] = xd[(jj * MB + mi + r * (MB / MT)) * WB + w];
#pragma unroll
      for (int c = 0; c < IT; ++c) wa[c] = wd[(jj * IB + ii + c * (IB / IT)) * WB + w];
#pragma unroll
      for (int r = 0; r < MT; ++r)
#pragma unroll
        for (int c = 0; c < IT; ++c) {
          acc[r][c].x = fmaf(xa[r].x, wa[c].x, acc[r][c].x);
          acc[r][c].x = fmaf(-xa[r].y, wa[c].y, acc[r][c].x);
          acc[r][c].y = fmaf(xa[r].x, wa[c].y, acc[r][c].y);
          acc[r][c].y = fmaf(xa[r].y, wa[c].x, acc[r][c].y);
        }
    }
    __syncthreads();
  }

  float2* Y = a.Y + wb * a.mstride * a.fo * WB;
#pragma unroll
  for (int r = 0; r < MT; ++r) {
    const int64_t m = m0 + mi + r * (MB / MT);
    if (m >= a.M) continue;
#pragma unroll
    for (int c = 0; c < IT; ++c) {
      const int i = i0 + ii + c * (IB / IT);
      if (i < a.fo) Y[(m * a.fo + i) * WB + w] = acc[r][c];
    }
  }
}

template <int T>
void fwd_t(Ctx* c, const FwdTileArgs& a, int64_t nblocks) {
  static bool configured = false;
  if (!configured) {
    VXG_CUDA_CHECK(cudaFuncSetAttribute(tile_fwd_kernel<T>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        TileCfg<T>::SMEM));
    configured = true;
  }
  tile_fwd_kernel<T><<<unsigned(nblocks), kFftThreads, TileCfg<T>::SMEM, c->stream>>>(a);
  c->counted();
  check_launch("tile_fwd_kernel");
}

template <int T>
void inv_t(Ctx* c, const InvTileArgs& a, int64_t nblocks) {
  static bool configured = false;
  if (!configured) {
    VXG_CUDA_CHECK(cudaFuncSetAttribute(tile_inv_kernel<T>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        TileCfg<T>::SMEM));
    configured = true;
  }
  tile_inv_kernel<T><<<unsigned(nblocks), kFftThreads, TileCfg<T>::SMEM, c->stream>>>(a);
  c->counted();
  check_launch("tile_inv_kernel");
}

template <int MT, int IT, int MB, int IB, int JC>
void gemm_t(Ctx* c, GemmArgs a, int64_t nwb) {
  using G = GemmCfg<MT, IT, MB, IB, JC>;
  static bool configured = false;
  if (!configured) {
    VXG_CUDA_CHECK(cudaFuncSetAttribute(cgemm_kernel<MT, IT, MB, IB, JC>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
    configured = true;
  }
  a.mblocks = int((a.M + MB - 1) / MB);
  a.iblocks = (a.fo + IB - 1) / IB;
  const int64_t blocks = int64_t(a.mblocks) * a.iblocks * nwb;
  require(blocks < (int64_t(1) << 31), "cgemm: grid too large");
  cgemm_kernel<MT, IT, MB, IB, JC><<<unsigned(blocks), G::THREADS, G::SMEM, c->stream>>>(a);
  c->counted();
  check_launch("cgemm_kernel");
}

}  // namespace

// supported tile FFT sizes (even, {2,3,5,7}-smooth)
const int kTileSizes[] = {4, 6, 8, 10, 12, 16, 20, 24, 28, 30, 32};
const int kNumTileSizes = sizeof(kTileSizes) / sizeof(int);

int64_t tile_nwb(int T) { return (int64_t(T) * T * (T / 2 + 1) + WB - 1) / WB; }

void launch_tile_fwd(Ctx* c, int T, const FwdTileArgs& a, int64_t nblocks) {
  const double nw = double(T) * T * (T / 2 + 1);
  KScope ks(c, a.kind, 0.0, double(nblocks) * (4.0 * double(T) * T * T + 8.0 * nw));
  switch (T) {
    case 4: fwd_t<4>(c, a, nblocks); break;
    case 6: fwd_t<6>(c, a, nblocks); break;
    case 8: fwd_t<8>(c, a, nblocks); break;
    case 10: fwd_t<10>(c, a, nblocks); break;
    case 12: fwd_t<12>(c, a, nblocks); break;
    case 16: fwd_t<16>(c, a, nblocks); break;
    case 20: fwd_t<20>(c, a, nblocks); break;
    case 24: fwd_t<24>(c, a, nblocks); break;
    case 28: fwd_t<28>(c, a, nblocks); break;
    case 30: fwd_t<30>(c, a, nblocks); break;
    case 32: fwd_t<32>(c, a, nblocks); break;
    default: throw invalid("tile fft: unsupported tile size");
  }
}

void launch_tile_inv(Ctx* c, int T, const InvTileArgs& a, int64_t nblocks) {
  const double nw = double(T) * T * (T / 2 + 1);
  KScope ks(c, VXG_K_TILE_INV, 0.0,
            double(nblocks) * (8.0 * nw + 4.0 * double(a.vx) * a.vy * a.vz));
  switch (T) {
    case 4: inv_t<4>(c, a, nblocks); break;
    case 6: inv_t<6>(c, a, nblocks); break;
    case 8: inv_t<8>(c, a, nblocks); break;
    case 10: inv_t<10>(c, a, nblocks); break;
    case 12: inv_t<12>(c, a, nblocks); break;
    case 16: inv_t<16>(c, a, nblocks); break;
    case 20: inv_t<20>(c, a, nblocks); break;
    case 24: inv_t<24>(c, a, nblocks); break;
    case 28: inv_t<28>(c, a, nblocks); break;
    case 30: inv_t<30>(c, a, nblocks); break;
    case 32: inv_t<32>(c, a, nblocks); break;
    default: throw invalid("tile fft: unsupported tile size");
  }
}

void launch_cgemm(Ctx* c, const GemmArgs& a, int64_t nwb) {
  const double nw = double(a.T) * a.T * (a.T / 2 + 1);  // true (unpadded) frequencies
  KScope ks(c, VXG_K_CGEMM, 8.0 * double(a.M) * a.f * a.fo * nw,
            8.0 * nw * (double(a.M) * a.f + double(a.M) * a.fo + double(a.f) * a.fo));
  if (a.fo >= 24)
    gemm_t<8, 5, 32, 40, 8>(c, a, nwb);
  else
    gemm_t<8, 2, 64, 4, 4>(c, a, nwb);
}

}  // namespace vxg
