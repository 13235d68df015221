// K3: per-frequency complex contraction of the tiled FFT convolution (fp32).
//
// The MAC loops of the reference (proj/include/voxin/layers.hpp:245-251,
// 330-344; task_conv.hpp:282-288), O[s,i](w) += I[s,j](w) * W[i,j](w), become
// for every frequency w a GEMM-shaped contraction over M = S * tiles rows:
//   Y[w](m, i) = sum_j X[w](m, j) W[w](i, j).
// CTA = 16 frequencies (one 128-byte spectrum line) x MB rows x IB output
// maps, all f input maps in JC-deep stages double-buffered with cp.async.
// Thread = one frequency x MT rows x IT maps (MT*IT complex accumulators,
// 4 FFMA per complex MAC).  Grid order keeps all m-blocks of one frequency
// block adjacent so the kernel-spectrum block stays L2-resident while X
// streams from HBM.
#include "async.cuh"
#include "common.cuh"
#include "fftconv.hpp"

namespace vxg {
namespace {

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

template <int MT, int IT, int MB, int IB, int JC>
void gemm_t(Ctx* c, GemmArgs a, int64_t nwb) {
  using G = GemmCfg<MT, IT, MB, IB, JC>;
  static PerDeviceOnce configured;
  if (configured.first()) {
    VXG_CUDA_CHECK(cudaFuncSetAttribute(cgemm_kernel<MT, IT, MB, IB, JC>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
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
