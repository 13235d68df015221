// Layer drivers: tile-size planning, kernel spectra, chunked FFT convolution
// and the direct path.  Chunking over (batch, tile) rows bounds the spectrum
// buffers under the HBM budget the same way sub_batch_limit bounds the
// reference's transform scratch (proj/include/voxin/fft.hpp:74-90).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>

#include "fftconv.hpp"

namespace vxg {

int64_t fft_chunk_bytes(const FftPlan& plan, int64_t f, int64_t fo, int64_t rows) {
  return rows * (f + fo) * plan.nwb * 16 * 8;
}

FftPlan plan_fft(V3 n, V3 k, int64_t f, int64_t fo, int64_t S, int T_forced) {
  FftPlan best;
  best.cost = std::numeric_limits<double>::infinity();
  const V3 no{n.x - k.x + 1, n.y - k.y + 1, n.z - k.z + 1};
  if (T_forced <= 0) {
    // experiment hook: VXG_FFT_TILE=<T> pins the tile size when it covers the kernel
    if (const char* env = std::getenv("VXG_FFT_TILE")) {
      const int t = std::atoi(env);
      if (t >= k.x && t >= k.y && t >= k.z) T_forced = t;
    }
  }
  for (int ti = 0; ti < kNumTileSizes; ++ti) {
    const int T = kTileSizes[ti];
    if (T_forced > 0 && T != T_forced) continue;
    if (T < k.x || T < k.y || T < k.z) continue;
    FftPlan p;
    p.T = T;
    for (int a = 0; a < 3; ++a) {
      p.v[a] = T - k[a] + 1;
      p.nt[a] = (no[a] + p.v[a] - 1) / p.v[a];
    }
    p.tiles = p.nt.vol();
    p.nwb = tile_nwb(T);
    const double M = double(S) * double(p.tiles);
    const double nw = double(p.nwb) * 16.0;
    // modelled seconds: contraction at ~50 TFLOP/s fp32, spectrum + image
    // traffic at ~5 TB/s, and a per-CTA transform overhead
    const double flops = 8.0 * M * double(f) * double(fo) * nw;
    const double bytes = M * (double(f) * (double(T) * T * T * 4.0 + 3.0 * nw * 8.0) +
                              double(fo) * (3.0 * nw * 8.0 + double(p.v.vol()) * 4.0));
    const double ctas = M * double(f + fo);
    p.cost = flops / 50e12 + bytes / 5e12 + ctas * (double(T) * T * T) * 2e-14 * std::log2(double(T));
    if (p.cost < best.cost) best = p;
  }
  if (best.T == 0) throw invalid("conv fft: no supported tile size covers the kernel");
  return best;
}

void compute_kernel_spectra(Ctx* c, int T, const float* w, int64_t fo, int64_t f, V3 k,
                            float2* out) {
  FwdTileArgs a{};
  a.src = w;
  a.img_stride = k.vol();
  a.nx = int(k.x); a.ny = int(k.y); a.nz = int(k.z);
  a.vx = a.vy = a.vz = 1;
  a.ntx = a.nty = a.ntz = 1;
  a.tiles_per_img = 1;
  a.f = f;
  a.m0 = 0;
  a.mstride = fo;
  a.out = out;
  a.scale = float(1.0 / (double(T) * double(T) * double(T)));
  a.kind = VXG_K_KSPEC;
  launch_tile_fwd(c, T, a, fo * f);
}

void conv_fft_device(Ctx* c, const float* in, int64_t S, int64_t f, V3 n, const float* w,
                     int64_t fo, V3 k, const float* bias, bool relu, float* out,
                     const FftPlan& plan, const float2* wspec, int64_t spectra_budget) {
  const V3 no{n.x - k.x + 1, n.y - k.y + 1, n.z - k.z + 1};
  const int T = plan.T;
  DevBuf wbuf;
  if (!wspec) {
    wbuf.alloc(c, plan.nwb * fo * f * 16 * 8);
    compute_kernel_spectra(c, T, w, fo, f, k, wbuf.as<float2>());
    wspec = wbuf.as<float2>();
  }
  const int64_t M = S * plan.tiles;
  const int64_t per_row = fft_chunk_bytes(plan, f, fo, 1);
  int64_t avail = spectra_budget;
  if (avail <= 0) {
    std::lock_guard<std::mutex> lk(c->mu);
    avail = int64_t(double(c->budget - c->current) * 0.95);
  }
  int64_t rows = std::max<int64_t>(1, avail / per_row);
  rows = std::min(rows, M);
  rows = std::min<int64_t>(rows, ((int64_t(1) << 31) - 1) / std::max(f, fo));
  DevBuf X(c, rows * f * plan.nwb * 16 * 8);
  DevBuf Y(c, rows * fo * plan.nwb * 16 * 8);

  for (int64_t m0 = 0; m0 < M; m0 += rows) {
    const int64_t mc = std::min(rows, M - m0);
    FwdTileArgs fa{};
    fa.src = in;
    fa.img_stride = n.vol();
    fa.nx = int(n.x); fa.ny = int(n.y); fa.nz = int(n.z);
    fa.vx = int(plan.v.x); fa.vy = int(plan.v.y); fa.vz = int(plan.v.z);
    fa.ntx = int(plan.nt.x); fa.nty = int(plan.nt.y); fa.ntz = int(plan.nt.z);
    fa.tiles_per_img = plan.tiles;
    fa.f = f;
    fa.m0 = m0;
    fa.mstride = rows;
    fa.out = X.as<float2>();
    fa.scale = 1.f;
    launch_tile_fwd(c, T, fa, mc * f);

    GemmArgs ga{};
    ga.X = X.as<float2>();
    ga.W = wspec;
    ga.Y = Y.as<float2>();
    ga.M = mc;
    ga.mstride = rows;
    ga.f = int(f);
    ga.fo = int(fo);
    ga.T = T;
    launch_cgemm(c, ga, plan.nwb);

    InvTileArgs ia{};
    ia.spec = Y.as<float2>();
    ia.mstride = rows;
    ia.fo = fo;
    ia.dst = out;
    ia.onx = int(no.x); ia.ony = int(no.y); ia.onz = int(no.z);
    ia.oel = no.vol();
    ia.vx = int(plan.v.x); ia.vy = int(plan.v.y); ia.vz = int(plan.v.z);
    ia.cx = int(k.x - 1); ia.cy = int(k.y - 1); ia.cz = int(k.z - 1);
    ia.ntx = int(plan.nt.x); ia.nty = int(plan.nt.y); ia.ntz = int(plan.nt.z);
    ia.tiles_per_img = plan.tiles;
    ia.m0 = m0;
    ia.bias = bias;
    ia.relu = relu ? 1 : 0;
    launch_tile_inv(c, T, ia, mc * fo);
  }
}

void conv_direct_device(Ctx* c, const float* in, int64_t S, int64_t f, V3 n, const float* w,
                        int64_t fo, V3 k, const float* bias, bool relu, float* out) {
  for (int64_t s0 = 0; s0 < S; s0 += 65535) {
    const int64_t sn = std::min<int64_t>(65535, S - s0);
    const V3 no{n.x - k.x + 1, n.y - k.y + 1, n.z - k.z + 1};
    launch_conv_direct(c, in + s0 * f * n.vol(), sn, f, n, w, fo, k, bias, relu,
                       out + s0 * fo * no.vol());
  }
}

}  // namespace vxg
