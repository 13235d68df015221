// Generic strided-line FFT and the reference-layout whole-image transforms.
//   pruned_forward_into      proj/include/voxin/fft.hpp:129-174
//   pruned_inverse_region    fft.hpp:181-228
//   batched_forward_into     fft.hpp:266-318
//   batched_inverse_region   fft.hpp:325-383
// These are the transform-level primitives of the public API (parity and
// tooling); the convolution hot path uses the on-chip tile transforms of
// k_fftconv.cu instead.
#include <cmath>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "linefft.hpp"

namespace vxg {
namespace {

constexpr int kMaxN = 2048;
constexpr int kLineThreads = 256;

struct LineJob {
  int N;
  int64_t nl1, nl2, nlines;     // line index = (i0, i1, i2), i1 < nl1, i2 < nl2
  const void* in;
  int in_real;                  // float input (else float2)
  int64_t in_s0, in_s1, in_s2, in_se;
  int in_count;                 // present elements (rest zero)
  int hermitian;                // input holds in_count = N/2+1 values of a real signal's spectrum
  void* out;
  int out_real;                 // write real parts (else float2)
  int64_t out_s0, out_s1, out_s2, out_se;
  int out_begin, out_count;
  float scale;
  int inverse;
  int nfactors;
  int factors[16];
  const float2* tw;             // W_N^t, t < N
};

__device__ __forceinline__ float2 tw_at(const float2* tw, int64_t e, int N, int inv) {
  const float2 w = tw[e % N];
  return inv ? make_float2(w.x, -w.y) : w;
}

__global__ void __launch_bounds__(kLineThreads) line_fft_kernel(LineJob j) {
  __shared__ float2 buf[2][kMaxN];
  const int64_t l = blockIdx.x;
  const int64_t i2 = l % j.nl2, i1 = (l / j.nl2) % j.nl1, i0 = l / (j.nl2 * j.nl1);
  const int N = j.N;
  // gather
  const int64_t ib = i0 * j.in_s0 + i1 * j.in_s1 + i2 * j.in_s2;
  for (int t = threadIdx.x; t < N; t += kLineThreads) {
    float2 v = make_float2(0.f, 0.f);
    if (j.hermitian) {
      const int k = t < j.in_count ? t : N - t;
      const float2 c = reinterpret_cast<const float2*>(j.in)[ib + int64_t(k) * j.in_se];
      v = t < j.in_count ? c : make_float2(c.x, -c.y);
    } else if (t < j.in_count) {
      if (j.in_real)
        v = make_float2(reinterpret_cast<const float*>(j.in)[ib + int64_t(t) * j.in_se], 0.f);
      else
        v = reinterpret_cast<const float2*>(j.in)[ib + int64_t(t) * j.in_se];
    }
    buf[0][t] = v;
  }
  __syncthreads();
  // Stockham autosort, radix stages in factor order
  int cur = 0;
  int Ns = 1;
  for (int fi = 0; fi < j.nfactors; ++fi) {
    const int R = j.factors[fi];
    const int NR = N / R;
    const int span = N / (Ns * R);
    for (int q = threadIdx.x; q < NR; q += kLineThreads) {
      float2 v[7];
      const int k = q % Ns;
      for (int r = 0; r < R; ++r) {
        const float2 x = buf[cur][q + r * NR];
        const float2 w = tw_at(j.tw, int64_t(r) * k * span, N, j.inverse);
        v[r] = make_float2(x.x * w.x - x.y * w.y, x.x * w.y + x.y * w.x);
      }
      float2 o[7];
      for (int kk = 0; kk < R; ++kk) {
        float2 acc = v[0];
        for (int r = 1; r < R; ++r) {
          const float2 w = tw_at(j.tw, int64_t(r) * kk * NR, N, j.inverse);
          acc.x += v[r].x * w.x - v[r].y * w.y;
          acc.y += v[r].x * w.y + v[r].y * w.x;
        }
        o[kk] = acc;
      }
      const int d = (q / Ns) * Ns * R + k;
      for (int r = 0; r < R; ++r) buf[cur ^ 1][d + r * Ns] = o[r];
    }
    __syncthreads();
    cur ^= 1;
    Ns *= R;
  }
  // scatter
  const int64_t ob = i0 * j.out_s0 + i1 * j.out_s1 + i2 * j.out_s2;
  for (int t = threadIdx.x; t < j.out_count; t += kLineThreads) {
    const float2 v = buf[cur][j.out_begin + t];
    if (j.out_real)
      reinterpret_cast<float*>(j.out)[ob + int64_t(t) * j.out_se] = v.x * j.scale;
    else
      reinterpret_cast<float2*>(j.out)[ob + int64_t(t) * j.out_se] =
          make_float2(v.x * j.scale, v.y * j.scale);
  }
}

std::mutex g_tw_mu;
std::map<std::pair<int, int>, float2*> g_tw;  // (device, N) -> table

const float2* twiddles(Ctx* c, int N) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto key = std::make_pair(c->device, N);
  auto it = g_tw.find(key);
  if (it != g_tw.end()) return it->second;
  std::vector<float2> h(static_cast<size_t>(N));
  for (int t = 0; t < N; ++t) {
    const double a = -2.0 * M_PI * double(t) / double(N);  // unit_roots, dft.hpp:39-47
    h[size_t(t)] = make_float2(float(std::cos(a)), float(std::sin(a)));
  }
  float2* d = nullptr;
  VXG_CUDA_CHECK(cudaMalloc(&d, sizeof(float2) * size_t(N)));
  VXG_CUDA_CHECK(cudaMemcpy(d, h.data(), sizeof(float2) * size_t(N), cudaMemcpyHostToDevice));
  g_tw[key] = d;
  return d;
}

void set_factors(LineJob& j) {
  int n = j.N, nf = 0;
  while (n % 4 == 0) { j.factors[nf++] = 4; n /= 4; }
  for (int p : {2, 3, 5, 7})
    while (n % p == 0) { j.factors[nf++] = p; n /= p; }
  if (n != 1) throw invalid("device transforms accept only sizes with prime factors {2,3,5,7}");
  j.nfactors = nf;
}

void run_lines(Ctx* c, LineJob j, int64_t n0) {
  require(j.N <= kMaxN, "device line transform longer than 2048");
  set_factors(j);
  j.tw = twiddles(c, j.N);
  j.nlines = n0 * j.nl1 * j.nl2;
  if (j.nlines == 0) return;
  require(j.nlines < (int64_t(1) << 31), "device line transform: too many lines");
  KScope ks(c, VXG_K_LINEFFT, 0.0, 16.0 * double(j.nlines) * j.N);
  line_fft_kernel<<<unsigned(j.nlines), kLineThreads, 0, c->stream>>>(j);
  c->counted();
  check_launch("line_fft_kernel");
}

LineJob job(int N) {
  LineJob j{};
  j.N = N;
  j.nl1 = j.nl2 = 1;
  j.scale = 1.f;
  return j;
}

}  // namespace

void init_line_fft(Ctx*) {}

// pruned_forward_into (fft.hpp:129-174): x r2c lines for the populated (y, z),
// y lines for the populated z, then every z line.  Spectrum (xh, py, pz).
void pruned_forward_device(Ctx* c, const float* img, V3 n, V3 p, float2* spec) {
  const int64_t xh = p.x / 2 + 1;
  VXG_CUDA_CHECK(cudaMemsetAsync(spec, 0, sizeof(float2) * size_t(xh * p.y * p.z), c->stream));
  LineJob a = job(int(p.x));
  a.in = img; a.in_real = 1; a.in_count = int(n.x);
  a.nl1 = n.y; a.nl2 = n.z; a.in_s1 = n.z; a.in_s2 = 1; a.in_se = n.y * n.z;
  a.out = spec; a.out_s1 = p.z; a.out_s2 = 1; a.out_se = p.y * p.z;
  a.out_begin = 0; a.out_count = int(xh);
  run_lines(c, a, 1);
  LineJob b = job(int(p.y));
  b.in = spec; b.in_count = int(p.y);
  b.nl1 = xh; b.nl2 = n.z; b.in_s1 = p.y * p.z; b.in_s2 = 1; b.in_se = p.z;
  b.out = spec; b.out_s1 = p.y * p.z; b.out_s2 = 1; b.out_se = p.z; b.out_count = int(p.y);
  run_lines(c, b, 1);
  LineJob z = job(int(p.z));
  z.in = spec; z.in_count = int(p.z);
  z.nl1 = xh; z.nl2 = p.y; z.in_s1 = p.y * p.z; z.in_s2 = p.z; z.in_se = 1;
  z.out = spec; z.out_s1 = p.y * p.z; z.out_s2 = p.z; z.out_se = 1; z.out_count = int(p.z);
  run_lines(c, z, 1);
}

// pruned_inverse_region (fft.hpp:181-228) with begin = 0: every z line, y lines
// for the crop's z, x lines (Hermitian completion) for the crop's (y, z).
void pruned_inverse_device(Ctx* c, const float2* spec_in, V3 p, V3 crop, float* out) {
  const int64_t xh = p.x / 2 + 1;
  DevBuf s(c, int64_t(sizeof(float2)) * xh * p.y * p.z);
  float2* spec = s.as<float2>();
  VXG_CUDA_CHECK(cudaMemcpyAsync(spec, spec_in, sizeof(float2) * size_t(xh * p.y * p.z),
                                 cudaMemcpyDeviceToDevice, c->stream));
  LineJob z = job(int(p.z));
  z.inverse = 1;
  z.in = spec; z.in_count = int(p.z);
  z.nl1 = xh; z.nl2 = p.y; z.in_s1 = p.y * p.z; z.in_s2 = p.z; z.in_se = 1;
  z.out = spec; z.out_s1 = p.y * p.z; z.out_s2 = p.z; z.out_se = 1; z.out_count = int(p.z);
  run_lines(c, z, 1);
  LineJob y = job(int(p.y));
  y.inverse = 1;
  y.in = spec; y.in_count = int(p.y);
  y.nl1 = xh; y.nl2 = crop.z; y.in_s1 = p.y * p.z; y.in_s2 = 1; y.in_se = p.z;
  y.out = spec; y.out_s1 = p.y * p.z; y.out_s2 = 1; y.out_se = p.z; y.out_count = int(p.y);
  run_lines(c, y, 1);
  LineJob x = job(int(p.x));
  x.inverse = 1;
  x.in = spec; x.hermitian = 1; x.in_count = int(xh);
  x.nl1 = crop.y; x.nl2 = crop.z; x.in_s1 = p.z; x.in_s2 = 1; x.in_se = p.y * p.z;
  x.out = out; x.out_real = 1; x.out_s1 = crop.z; x.out_s2 = 1; x.out_se = crop.y * crop.z;
  x.out_begin = 0; x.out_count = int(crop.x);
  x.scale = float(1.0 / (double(p.x) * double(p.y) * double(p.z)));
  run_lines(c, x, 1);
}

// batched_forward_into (fft.hpp:266-318): z r2c lines of every (b, x, y),
// then y lines of the populated x, then all x lines; result (b, zh, py, px).
void batched_forward_device(Ctx* c, const float* imgs, int64_t b, V3 n, V3 p, float2* spec) {
  const int64_t zh = p.z / 2 + 1;
  const int64_t S = zh * p.y * p.x;
  VXG_CUDA_CHECK(cudaMemsetAsync(spec, 0, sizeof(float2) * size_t(b * S), c->stream));
  LineJob a = job(int(p.z));
  a.in = imgs; a.in_real = 1; a.in_count = int(n.z);
  a.nl1 = n.x; a.nl2 = n.y; a.in_s0 = n.vol(); a.in_s1 = n.y * n.z; a.in_s2 = n.z; a.in_se = 1;
  a.out = spec; a.out_s0 = S; a.out_s1 = 1; a.out_s2 = p.x; a.out_se = p.y * p.x;
  a.out_begin = 0; a.out_count = int(zh);
  run_lines(c, a, b);
  LineJob y = job(int(p.y));
  y.in = spec; y.in_count = int(p.y);
  y.nl1 = zh; y.nl2 = n.x; y.in_s0 = S; y.in_s1 = p.y * p.x; y.in_s2 = 1; y.in_se = p.x;
  y.out = spec; y.out_s0 = S; y.out_s1 = p.y * p.x; y.out_s2 = 1; y.out_se = p.x; y.out_count = int(p.y);
  run_lines(c, y, b);
  LineJob x = job(int(p.x));
  x.in = spec; x.in_count = int(p.x);
  x.nl1 = zh; x.nl2 = p.y; x.in_s0 = S; x.in_s1 = p.y * p.x; x.in_s2 = p.x; x.in_se = 1;
  x.out = spec; x.out_s0 = S; x.out_s1 = p.y * p.x; x.out_s2 = p.x; x.out_se = 1; x.out_count = int(p.x);
  run_lines(c, x, b);
}

// batched_inverse_region (fft.hpp:325-383) with begin = 0: every x line, y
// lines of the crop's x, z c2r lines (Hermitian completion) of the crop's (x, y).
void batched_inverse_device(Ctx* c, const float2* spec_in, int64_t b, V3 p, V3 crop, float* out) {
  const int64_t zh = p.z / 2 + 1;
  const int64_t S = zh * p.y * p.x;
  DevBuf s(c, int64_t(sizeof(float2)) * b * S);
  float2* spec = s.as<float2>();
  VXG_CUDA_CHECK(cudaMemcpyAsync(spec, spec_in, sizeof(float2) * size_t(b * S),
                                 cudaMemcpyDeviceToDevice, c->stream));
  LineJob x = job(int(p.x));
  x.inverse = 1;
  x.in = spec; x.in_count = int(p.x);
  x.nl1 = zh; x.nl2 = p.y; x.in_s0 = S; x.in_s1 = p.y * p.x; x.in_s2 = p.x; x.in_se = 1;
  x.out = spec; x.out_s0 = S; x.out_s1 = p.y * p.x; x.out_s2 = p.x; x.out_se = 1; x.out_count = int(p.x);
  run_lines(c, x, b);
  LineJob y = job(int(p.y));
  y.inverse = 1;
  y.in = spec; y.in_count = int(p.y);
  y.nl1 = zh; y.nl2 = crop.x; y.in_s0 = S; y.in_s1 = p.y * p.x; y.in_s2 = 1; y.in_se = p.x;
  y.out = spec; y.out_s0 = S; y.out_s1 = p.y * p.x; y.out_s2 = 1; y.out_se = p.x; y.out_count = int(p.y);
  run_lines(c, y, b);
  LineJob z = job(int(p.z));
  z.inverse = 1;
  z.in = spec; z.hermitian = 1; z.in_count = int(zh);
  z.nl1 = crop.x; z.nl2 = crop.y; z.in_s0 = S; z.in_s1 = 1; z.in_s2 = p.x; z.in_se = p.y * p.x;
  z.out = out; z.out_real = 1; z.out_s0 = crop.vol(); z.out_s1 = crop.y * crop.z; z.out_s2 = crop.z;
  z.out_se = 1; z.out_begin = 0; z.out_count = int(crop.z);
  z.scale = float(1.0 / (double(p.x) * double(p.y) * double(p.z)));
  run_lines(c, z, b);
}

}  // namespace vxg
