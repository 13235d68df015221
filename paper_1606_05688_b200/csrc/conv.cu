// Layer drivers: tile-size planning, kernel spectra, chunked FFT convolution
// and the direct path.  Chunking over (batch, tile) rows bounds the spectrum
// buffers under the HBM budget the same way sub_batch_limit bounds the
// reference's transform scratch (proj/include/voxin/fft.hpp:74-90).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>

#include "fftconv.hpp"

namespace vxg {

namespace {

// VXG_NO_TC=1 pins the fp32 FFMA contraction (parity cross-checks, A/B timing)
// VXG_YPAIR=1: pair-major Y (whole-line epilogue stores, TMA-gathered inverse).
// Measured at T = 32: contraction -33 %, inverse +110 % -> off by default.
bool ypair_enabled() {
  const char* e = std::getenv("VXG_YPAIR");
  return e && std::strcmp(e, "1") == 0;
}

// VXG_NO_FUSED_F1=1: single-input-map layers go through Y like the others
bool fused_f1_enabled() {
  const char* e = std::getenv("VXG_NO_FUSED_F1");
  return !(e && std::strcmp(e, "0") != 0);
}

bool tc_disabled() {
  const char* e = std::getenv("VXG_NO_TC");
  return e && std::strcmp(e, "0") != 0;
}

}  // namespace

bool trace_on() {
  static const bool on = [] {
    const char* e = std::getenv("VXG_TRACE");
    return e && std::strcmp(e, "0") != 0;
  }();
  return on;
}

int64_t fft_reserved_rows() {
  static const int64_t r = [] {
    const char* e = std::getenv("VXG_FFT_ROWS");
    const long long v = e ? std::atoll(e) : 0;
    return v > 0 ? int64_t(v) : int64_t(256);
  }();
  return r;
}

int64_t fft_chunk_bytes(const FftPlan& plan, int64_t f, int64_t fo, int64_t rows) {
  return rows * (plan.fused_f1 ? f : f + fo) * plan.nwp * 8;
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
  const bool tc = cgemm_tc_supported(f, fo) && !tc_disabled();
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
    p.lw = 16;
    p.tc = tc;
    p.quad = tc_quad_enabled();
    // measured wins: pairs at T = 24 / 32; one CTA at the other sizes it fits,
    // T = 36 included (199 KB of shared memory, one CTA per SM: 1.31 vs 1.44 ns
    // per output voxel on the CTA pair for 80 -> 80 k7, profiles/r2_experiments.md
    // §15); T = 40 exceeds one CTA's shared memory and runs on pairs only
    p.pair = ((T == 32 || T == 24) && tile_pair_enabled()) || T >= 40;
    p.inv_pair = ((T == 32 || T == 24) && tile_pair_enabled() && inv_pair_enabled()) || T >= 40;
    p.ylw = (tc && p.inv_pair && ypair_enabled()) ? 2 : 16;
    p.nwp = tile_nwp(T, p.lw);
    p.fused_f1 = f == 1 && !p.tc && fused_f1_enabled();
    const double M = double(S) * double(p.tiles);
    const double nw = double(T) * T * (T / 2 + 1);
    // Modelled seconds (calibrated on B200 with tools/kbench.py): the
    // contraction at ~40 TFLOP/s (FFMA) or ~150 TFLOP/s (tcgen05), the
    // transforms at ~140 ns per (tile, channel) CTA for T = 32 scaling with
    // T^3 log T, and the spectrum round trips at ~5 TB/s.
    const double flops = 8.0 * M * double(f) * double(fo) * nw;
    const double cta = 140e-9 * std::pow(double(T) / 32.0, 3.0) * std::log2(double(T)) / 5.0;
    const double bytes = 16.0 * M * double(f + fo) * nw;
    // T = 36 (one CTA) / 40 (CTA pairs) run one CTA per SM: measured ~1.5x the
    // per-(tile, channel) time the T^3 log T scaling predicts
    const double big = T >= 36 ? 1.5 : 1.0;
    p.cost = flops / (tc ? 150e12 : 40e12) + M * double(f + fo) * cta * big + bytes / 5e12;
    if (p.cost < best.cost) best = p;
  }
  if (best.T == 0) throw invalid("conv fft: no supported tile size covers the kernel");
  return best;
}

FftPlan plan_fft_forced(V3 n, V3 k, int64_t f, int64_t fo, int64_t S, int T, bool tc, bool pair) {
  FftPlan p = plan_fft(n, k, f, fo, S, T);
  if (p.T != T) throw invalid("conv fft: unsupported tile size");
  p.tc = tc && cgemm_tc_supported(f, fo);
  p.quad = tc_quad_enabled();
  p.pair = pair && T >= 24;  // tests: every pair-capable size
  p.inv_pair = pair && T >= 24;  // tests: every pair-capable size
  p.lw = 16;
  p.ylw = (p.tc && p.inv_pair && ypair_enabled()) ? 2 : 16;
  p.nwp = tile_nwp(T, p.lw);
  p.fused_f1 = f == 1 && !p.tc && fused_f1_enabled();
  return p;
}

int64_t kernel_spectra_bytes(const FftPlan& plan, int64_t f, int64_t fo) {
  if (plan.tc) return tc_wsplit_bytes(plan.nwp / 2, f, fo, plan.quad);
  return plan.nwp * fo * f * 8;
}

// tc: the raw spectra go through a scratch buffer and are stored pre-split
// for the tensor cores (tc_wsplit); otherwise raw into `out`.
void compute_kernel_spectra(Ctx* c, int T, bool tc, bool quad, const float* w, int64_t fo, int64_t f, V3 k,
                            float2* out) {
  DevBuf raw;
  float2* dst = out;
  if (tc) {
    raw.alloc(c, tile_nwp(T, 16) * fo * f * 8);
    dst = raw.as<float2>();
  }
  FwdTileArgs a{};
  a.src = w;
  a.img_stride = k.vol();
  a.nx = int(k.x); a.ny = int(k.y); a.nz = int(k.z);
  a.pz = int(k.z);
  a.vx = a.vy = a.vz = 1;
  a.ntx = a.nty = a.ntz = 1;
  a.tiles_per_img = 1;
  a.f = f;
  a.m0 = 0;
  a.mstride = fo;
  a.out = dst;
  a.scale = float(1.0 / (double(T) * double(T) * double(T)));
  a.kind = VXG_K_KSPEC;
  a.lw = 16;
  launch_tile_fwd(c, T, a, fo * f);
  if (tc) tc_wsplit(c, dst, out, tile_nwp(T, 16) / 2, f, fo, quad);
}

int64_t conv_fft_device(Ctx* c, const float* in, int64_t S, int64_t f, V3 n, const float* w,
                        int64_t fo, V3 k, const float* bias, bool relu, float* out,
                        const FftPlan& plan, const float2* wspec, int64_t spectra_budget, int64_t ipz,
                        int64_t opz) {
  const V3 no{n.x - k.x + 1, n.y - k.y + 1, n.z - k.z + 1};
  if (ipz <= 0) ipz = n.z;
  if (opz <= 0) opz = no.z;
  const int T = plan.T;
  DevBuf wbuf;
  if (!wspec) {
    wbuf.alloc(c, kernel_spectra_bytes(plan, f, fo));
    compute_kernel_spectra(c, T, plan.tc, plan.quad, w, fo, f, k, wbuf.as<float2>());
    wspec = wbuf.as<float2>();
  }
  const int64_t M = S * plan.tiles;
  const int64_t per_row = fft_chunk_bytes(plan, f, fo, 1);
  int64_t avail = spectra_budget;
  if (avail <= 0) avail = int64_t(double(c->avail()) * 0.98);
  int64_t rows = std::max<int64_t>(1, avail / per_row);
  rows = std::min(rows, M);
  rows = std::min<int64_t>(rows, ((int64_t(1) << 31) - 1) / std::max(f, fo));
  // Chunks of at most ~2048 rows: launches over 8000 rows (38 GB spectrum
  // buffers at T = 24) alternated between full speed and half speed in the
  // contraction from one identical launch to the next, while the same rows in
  // four chunks ran at full speed every time (profiles/r2_experiments.md §8);
  // the extra kernel-spectrum reads cost ~2 %.  VXG_MAX_ROWS overrides (0: none).
  static const int64_t max_rows = [] {
    const char* e = std::getenv("VXG_MAX_ROWS");
    return e ? int64_t(std::atoll(e)) : int64_t(2048);
  }();
  if (max_rows > 0 && rows > max_rows) rows = max_rows;
  {
    const int64_t nchunks = (M + rows - 1) / rows;
    rows = (M + nchunks - 1) / nchunks;  // balanced chunks
  }
  if (trace_on())
    std::fprintf(stderr, "[vxg] conv_fft S=%lld f=%lld fo=%lld n=%lld T=%d tiles=%lld M=%lld rows=%lld tc=%d\n",
                 (long long)S, (long long)f, (long long)fo, (long long)n.x, T, (long long)plan.tiles,
                 (long long)M, (long long)rows, int(plan.tc));
  DevBuf X(c, rows * f * plan.nwp * 8);
  DevBuf Ybuf;
  if (!plan.fused_f1) Ybuf.alloc(c, rows * fo * plan.nwp * 8);
  const DevBuf& Y = Ybuf;

  for (int64_t m0 = 0; m0 < M; m0 += rows) {
    const int64_t mc = std::min(rows, M - m0);
    FwdTileArgs fa{};
    fa.src = in;
    fa.img_stride = n.x * n.y * ipz;
    fa.nx = int(n.x); fa.ny = int(n.y); fa.nz = int(n.z);
    fa.pz = int(ipz);
    fa.vx = int(plan.v.x); fa.vy = int(plan.v.y); fa.vz = int(plan.v.z);
    fa.ntx = int(plan.nt.x); fa.nty = int(plan.nt.y); fa.ntz = int(plan.nt.z);
    fa.tiles_per_img = plan.tiles;
    fa.f = f;
    fa.m0 = m0;
    fa.mstride = rows;
    fa.out = X.as<float2>();
    fa.scale = 1.f;
    fa.lw = plan.lw;
    fa.pair = plan.pair;
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
    ga.ypair = plan.ylw == 2 ? 1 : 0;
    ga.quad = plan.quad ? 1 : 0;
    if (plan.fused_f1) {
      // the contraction is elementwise (one input map): done in the inverse's loads
    } else if (plan.tc) {
      launch_cgemm_tc(c, ga, plan.nwp / 2);
    } else {
      launch_cgemm(c, ga, plan.nwp / 16);
    }

    InvTileArgs ia{};
    ia.spec = Y.as<float2>();
    ia.mstride = rows;
    ia.fo = fo;
    ia.dst = out;
    ia.onx = int(no.x); ia.ony = int(no.y); ia.onz = int(no.z);
    ia.opz = int(opz);
    ia.oel = no.x * no.y * opz;
    ia.vx = int(plan.v.x); ia.vy = int(plan.v.y); ia.vz = int(plan.v.z);
    ia.cx = int(k.x - 1); ia.cy = int(k.y - 1); ia.cz = int(k.z - 1);
    ia.ntx = int(plan.nt.x); ia.nty = int(plan.nt.y); ia.ntz = int(plan.nt.z);
    ia.tiles_per_img = plan.tiles;
    ia.m0 = m0;
    ia.bias = bias;
    ia.relu = relu ? 1 : 0;
    ia.lw = plan.ylw;
    ia.nwp = plan.nwp;
    ia.pair = plan.inv_pair;
    if (plan.fused_f1) {
      ia.spec = X.as<float2>();
      ia.wsp = wspec;
      ia.w_fo = fo;
    }
    launch_tile_inv(c, T, ia, mc * fo);
  }
  return rows;
}

void conv_direct_device(Ctx* c, const float* in, int64_t S, int64_t f, V3 n, const float* w,
                        int64_t fo, V3 k, const float* bias, bool relu, float* out, int64_t ipz,
                        int64_t opz) {
  const V3 no{n.x - k.x + 1, n.y - k.y + 1, n.z - k.z + 1};
  if (ipz <= 0) ipz = n.z;
  if (opz <= 0) opz = no.z;
  for (int64_t s0 = 0; s0 < S; s0 += 65535) {
    const int64_t sn = std::min<int64_t>(65535, S - s0);
    launch_conv_direct(c, in + s0 * f * n.x * n.y * ipz, sn, f, n, w, fo, k, bias, relu,
                       out + s0 * fo * no.x * no.y * opz, ipz, opz);
  }
}

}  // namespace vxg
