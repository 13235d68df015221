// Register-resident mixed-radix FFTs of compile-time length N (radices
// 4, 2, 3, 5, 7), fully unrolled.  Twiddles W_N^t = exp(-2 pi i t / N) are
// computed in double on the host (as unit_roots, proj/include/voxin/dft.hpp:
// 39-47) and read from constant memory at compile-time offsets, so every
// twiddle is an immediate constant-bank operand.  The 1D engine contract of
// Dft1d (dft.hpp:15-25) holds: forward uses W, inverse uses conj(W), and the
// inverse is unnormalised.
#pragma once

#include <cuda_runtime.h>

namespace vxg {
namespace fftreg {

// every size a tile transform may use (all {2,3,5,7}-smooth sizes <= 64)
constexpr int kSizes[] = {1,  2,  3,  4,  5,  6,  7,  8,  9,  10, 12, 14, 15, 16, 18, 20, 21, 24,
                          25, 27, 28, 30, 32, 35, 36, 40, 42, 45, 48, 49, 50, 54, 56, 60, 63, 64};
constexpr int kNumSizes = sizeof(kSizes) / sizeof(int);

constexpr int tw_offset(int n) {
  int off = 0;
  for (int i = 0; i < kNumSizes; ++i) {
    if (kSizes[i] == n) return off;
    off += kSizes[i];
  }
  return -1;
}
constexpr int kTwTotal = tw_offset(64) + 64;

constexpr int radix_of(int n) {
  return n % 4 == 0 ? 4 : (n % 2 == 0 ? 2 : (n % 3 == 0 ? 3 : (n % 5 == 0 ? 5 : 7)));
}

}  // namespace fftreg

// defined here: this header is included by exactly one translation unit
// (k_fftconv.cu), which also uploads the table (init_twiddles)
__constant__ float2 c_twiddle[fftreg::kTwTotal];

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

// W_N^e (e reduced mod N at compile time after unrolling)
template <int N, bool INV>
__device__ __forceinline__ float2 tw(int e) {
  const float2 w = c_twiddle[fftreg::tw_offset(N) + (e % N)];
  return INV ? cconj(w) : w;
}

// multiply by W_N^e, skipping the exact unit cases that unrolling exposes
template <int N, bool INV>
__device__ __forceinline__ float2 twmul(float2 a, int e) {
  e %= N;
  if (e == 0) return a;
  if (4 * e == N) return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);      // -i / +i
  if (2 * e == N) return make_float2(-a.x, -a.y);
  if (4 * e == 3 * N) return INV ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
  return cmul(a, tw<N, INV>(e));
}

// Small DFT of length R in place on t[0..R).
template <int R, bool INV>
__device__ __forceinline__ void small_dft(float2 (&t)[R]) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    const float2 a = t[0], b = t[1];
    t[0] = cadd(a, b);
    t[1] = csub(a, b);
  } else if constexpr (R == 3) {
    // X0 = x0 + t1, X1/2 = x0 - t1/2 -/+ i s (x1 - x2), s = sin(2 pi / 3) (forward)
    constexpr float s = 0.866025403784438647f;
    const float2 t1 = cadd(t[1], t[2]), d = csub(t[1], t[2]);
    const float2 m = make_float2(fmaf(-0.5f, t1.x, t[0].x), fmaf(-0.5f, t1.y, t[0].y));
    const float2 r = INV ? make_float2(-s * d.y, s * d.x) : make_float2(s * d.y, -s * d.x);
    t[0] = cadd(t[0], t1);
    t[1] = cadd(m, r);
    t[2] = csub(m, r);
  } else if constexpr (R == 5) {
    // Winograd-style 5-point DFT: a_k = x0 + c.(x1+x4) + c'.(x2+x3),
    // b_k = s.(x1-x4) + s'.(x2-x3); X_k = a_k -/+ i b_k (forward / inverse)
    constexpr float c1 = 0.309016994374947424f, c2 = -0.809016994374947424f;
    constexpr float s1 = 0.951056516295153572f, s2 = 0.587785252292473129f;
    const float2 t1 = cadd(t[1], t[4]), t2 = cadd(t[2], t[3]);
    const float2 t3 = csub(t[1], t[4]), t4 = csub(t[2], t[3]);
    const float2 a1 = make_float2(fmaf(c1, t1.x, fmaf(c2, t2.x, t[0].x)), fmaf(c1, t1.y, fmaf(c2, t2.y, t[0].y)));
    const float2 a2 = make_float2(fmaf(c2, t1.x, fmaf(c1, t2.x, t[0].x)), fmaf(c2, t1.y, fmaf(c1, t2.y, t[0].y)));
    const float2 b1 = make_float2(fmaf(s1, t3.x, s2 * t4.x), fmaf(s1, t3.y, s2 * t4.y));
    const float2 b2 = make_float2(fmaf(s2, t3.x, -s1 * t4.x), fmaf(s2, t3.y, -s1 * t4.y));
    // -i b = (b.y, -b.x); +i b = (-b.y, b.x)
    const float2 nb1 = INV ? make_float2(-b1.y, b1.x) : make_float2(b1.y, -b1.x);
    const float2 nb2 = INV ? make_float2(-b2.y, b2.x) : make_float2(b2.y, -b2.x);
    t[0] = cadd(t[0], cadd(t1, t2));
    t[1] = cadd(a1, nb1);
    t[4] = csub(a1, nb1);
    t[2] = cadd(a2, nb2);
    t[3] = csub(a2, nb2);
  } else if constexpr (R == 4) {
    const float2 a0 = cadd(t[0], t[2]), a1 = csub(t[0], t[2]);
    const float2 b0 = cadd(t[1], t[3]), b1 = csub(t[1], t[3]);
    // b1 * (-i) forward, (+i) inverse
    const float2 jb1 = INV ? make_float2(-b1.y, b1.x) : make_float2(b1.y, -b1.x);
    t[0] = cadd(a0, b0);
    t[2] = csub(a0, b0);
    t[1] = cadd(a1, jb1);
    t[3] = csub(a1, jb1);
  } else {
    float2 o[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      float2 acc = t[0];
#pragma unroll
      for (int q = 1; q < R; ++q) acc = cadd(acc, twmul<R, INV>(t[q], q * k));
      o[k] = acc;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) t[k] = o[k];
  }
}

// In-register DFT of length N: x[k] = sum_j x[j] W_N^{jk} (decimation in time).
template <int N, bool INV>
__device__ __forceinline__ void fft(float2 (&x)[N]) {
  if constexpr (N == 1) {
  } else if constexpr (N == 2 || N == 3 || N == 4 || N == 5 || N == 7) {
    small_dft<N, INV>(x);
  } else {
    constexpr int R = fftreg::radix_of(N);
    constexpr int M = N / R;
    float2 sub[R][M];
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
      for (int j = 0; j < M; ++j) sub[q][j] = x[q + R * j];
#pragma unroll
    for (int q = 0; q < R; ++q) fft<M, INV>(sub[q]);
#pragma unroll
    for (int k1 = 0; k1 < M; ++k1) {
      float2 t[R];
#pragma unroll
      for (int q = 0; q < R; ++q) t[q] = twmul<N, INV>(sub[q][k1], q * k1);
      small_dft<R, INV>(t);
#pragma unroll
      for (int k2 = 0; k2 < R; ++k2) x[k1 + M * k2] = t[k2];
    }
  }
}

}  // namespace vxg
