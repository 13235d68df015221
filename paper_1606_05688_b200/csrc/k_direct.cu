// K5: direct 3D convolution, fp32 FFMA, register-tiled.
//
//   conv_direct / accumulate_valid_conv  proj/include/voxin/layers.hpp:120-192
//   out[s,j,p] = act(bias[j] + sum_i sum_q w[j,i,q] * in[s,i,p+k-1-q])
//
// CTA tile: 4 (x) x 8 (y) x 32 (z) output voxels x 16 output maps; each of the
// 256 threads owns 4 consecutive z outputs x 16 maps (64 accumulators).  Per
// input map the CTA stages the (4+kx-1)(8+ky-1)(32+kz-1) input box and the
// 16 x k^3 weights in shared memory; weights are laid out [q][j] so one
// broadcast LDS.128 feeds 4 maps.  The kz loop is unrolled by template.
// This is the planner's choice for the f=1 first layer of every bundled net
// (small k, tiny f), where the FFT's transform traffic cannot amortise.
#include "common.cuh"

namespace vxg {
namespace {

constexpr int TX = 4, TY = 8, TZ = 32, ZR = 4, JB = 16;
constexpr int THREADS = (TX * TY * TZ) / ZR;  // 256

struct DirectGeom {
  int64_t S, f, fo;
  int nx, ny, nz;
  int kx, ky, kz;
  int ox, oy, oz;           // output extents
  int ipz, opz;             // z row pitch of input / output
  int tiles_x, tiles_y, tiles_z;
  int relu;
};

template <int KZ>
__global__ void __launch_bounds__(THREADS) conv_direct_kernel(const float* __restrict__ in,
                                                              const float* __restrict__ w,
                                                              const float* __restrict__ bias,
                                                              float* __restrict__ out,
                                                              DirectGeom g) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int kz = KZ > 0 ? KZ : g.kz;
  const int kvol = g.kx * g.ky * kz;
  const int bx = TX + g.kx - 1, by = TY + g.ky - 1, bz = TZ + kz - 1;
  float* ws = smem;                              // [kvol][JB]
  float* is = smem + kvol * JB;                  // [bx][by][bz]

  const int tile = blockIdx.x;
  const int tz0 = (tile % g.tiles_z) * TZ;
  const int ty0 = ((tile / g.tiles_z) % g.tiles_y) * TY;
  const int tx0 = (tile / (g.tiles_z * g.tiles_y)) * TX;
  const int j0 = blockIdx.y * JB;
  const int64_t s = blockIdx.z;

  const int tid = threadIdx.x;
  const int lz = (tid % (TZ / ZR)) * ZR;
  const int ly = (tid / (TZ / ZR)) % TY;
  const int lx = tid / ((TZ / ZR) * TY);

  float acc[JB][ZR];
#pragma unroll
  for (int j = 0; j < JB; ++j)
#pragma unroll
    for (int r = 0; r < ZR; ++r) acc[j][r] = 0.f;

  const int64_t nel = int64_t(g.nx) * g.ny * g.ipz;
  for (int64_t i = 0; i < g.f; ++i) {
    __syncthreads();
    // weights of maps j0..j0+15 for input map i, transposed to [q][j]
    for (int t = tid; t < kvol * JB; t += THREADS) {
      const int j = t % JB, q = t / JB;
      ws[t] = (j0 + j < g.fo) ? __ldg(w + ((j0 + j) * g.f + i) * int64_t(kvol) + q) : 0.f;
    }
    // input box, zero outside the image
    const float* src = in + (s * g.f + i) * nel;
    const int box = bx * by * bz;
    for (int t = tid; t < box; t += THREADS) {
      const int zz = t % bz, yy = (t / bz) % by, xx = t / (bz * by);
      const int gx = tx0 + xx, gy = ty0 + yy, gz = tz0 + zz;
      float v = 0.f;
      if (gx < g.nx && gy < g.ny && gz < g.nz) v = __ldg(src + (int64_t(gx) * g.ny + gy) * g.ipz + gz);
      is[t] = v;
    }
    __syncthreads();
    for (int qx = 0; qx < g.kx; ++qx)
      for (int qy = 0; qy < g.ky; ++qy) {
        // in[p + k - 1 - q]: box coordinates (lx + kx-1-qx, ly + ky-1-qy, lz + kz-1-qz)
        const float* row = is + ((lx + g.kx - 1 - qx) * by + (ly + g.ky - 1 - qy)) * bz + lz;
        float rv[ZR + (KZ > 0 ? KZ : 16) - 1];
        if (KZ > 0) {
#pragma unroll
          for (int r = 0; r < ZR + KZ - 1; ++r) rv[r] = row[r];
#pragma unroll
          for (int qz = 0; qz < KZ; ++qz) {
            const float4* wq = reinterpret_cast<const float4*>(ws + ((qx * g.ky + qy) * KZ + qz) * JB);
#pragma unroll
            for (int j4 = 0; j4 < JB / 4; ++j4) {
              const float4 wv = wq[j4];
#pragma unroll
              for (int r = 0; r < ZR; ++r) {
                const float iv = rv[r + KZ - 1 - qz];
                acc[4 * j4 + 0][r] = fmaf(wv.x, iv, acc[4 * j4 + 0][r]);
                acc[4 * j4 + 1][r] = fmaf(wv.y, iv, acc[4 * j4 + 1][r]);
                acc[4 * j4 + 2][r] = fmaf(wv.z, iv, acc[4 * j4 + 2][r]);
                acc[4 * j4 + 3][r] = fmaf(wv.w, iv, acc[4 * j4 + 3][r]);
              }
            }
          }
        } else {
          for (int qz = 0; qz < kz; ++qz) {
            const float4* wq = reinterpret_cast<const float4*>(ws + ((qx * g.ky + qy) * kz + qz) * JB);
#pragma unroll
            for (int j4 = 0; j4 < JB / 4; ++j4) {
              const float4 wv = wq[j4];
#pragma unroll
              for (int r = 0; r < ZR; ++r) {
                const float iv = row[r + kz - 1 - qz];
                acc[4 * j4 + 0][r] = fmaf(wv.x, iv, acc[4 * j4 + 0][r]);
                acc[4 * j4 + 1][r] = fmaf(wv.y, iv, acc[4 * j4 + 1][r]);
                acc[4 * j4 + 2][r] = fmaf(wv.z, iv, acc[4 * j4 + 2][r]);
                acc[4 * j4 + 3][r] = fmaf(wv.w, iv, acc[4 * j4 + 3][r]);
              }
            }
          }
        }
      }
  }

  const int gx = tx0 + lx, gy = ty0 + ly;
  if (gx >= g.ox || gy >= g.oy) return;
  const int64_t oel = int64_t(g.ox) * g.oy * g.opz;
#pragma unroll
  for (int j = 0; j < JB; ++j) {
    if (j0 + j >= g.fo) break;
    const float b = __ldg(bias + j0 + j);
    float* o = out + (s * g.fo + j0 + j) * oel + (int64_t(gx) * g.oy + gy) * g.opz;
#pragma unroll
    for (int r = 0; r < ZR; ++r) {
      const int gz = tz0 + lz + r;
      if (gz < g.oz) {
        const float v = acc[j][r] + b;
        o[gz] = g.relu ? (v > 0.f ? v : 0.f) : v;  // activate (layers.hpp:105-108)
      }
    }
  }
}

template <int KZ>
void run_direct(Ctx* c, const float* in, const float* w, const float* bias, float* out,
                const DirectGeom& g) {
  const int kz = KZ > 0 ? KZ : g.kz;
  const int kvol = g.kx * g.ky * kz;
  const size_t smem = sizeof(float) * (size_t(kvol) * JB +
                                       size_t(TX + g.kx - 1) * (TY + g.ky - 1) * (TZ + kz - 1));
  require(smem <= 200 * 1024, "conv_direct: kernel too large for the direct device kernel");
  static PerDeviceOnce configured;
  if (configured.first()) {
    VXG_CUDA_CHECK(cudaFuncSetAttribute(conv_direct_kernel<KZ>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  }
  dim3 grid(unsigned(g.tiles_x) * g.tiles_y * g.tiles_z, unsigned((g.fo + JB - 1) / JB),
            unsigned(g.S));
  const double vox = double(g.ox) * g.oy * g.oz;
  KScope ks(c, VXG_K_DIRECT, 2.0 * double(g.S) * g.f * g.fo * vox * double(kvol),
            4.0 * (double(g.S) * g.f * g.nx * g.ny * g.nz + double(g.S) * g.fo * vox +
                   double(g.fo) * g.f * kvol));
  conv_direct_kernel<KZ><<<grid, THREADS, smem, c->stream>>>(in, w, bias, out, g);
  c->counted();
  check_launch("conv_direct_kernel");
}

}  // namespace

void launch_conv_direct(Ctx* c, const float* in, i64 S, i64 f, V3 n, const float* w, i64 fo,
                        V3 k, const float* bias, bool relu, float* out, i64 ipz, i64 opz) {
  DirectGeom g{};
  g.S = S; g.f = f; g.fo = fo;
  g.nx = int(n.x); g.ny = int(n.y); g.nz = int(n.z);
  g.kx = int(k.x); g.ky = int(k.y); g.kz = int(k.z);
  g.ox = int(n.x - k.x + 1); g.oy = int(n.y - k.y + 1); g.oz = int(n.z - k.z + 1);
  g.ipz = int(ipz > 0 ? ipz : n.z);
  g.opz = int(opz > 0 ? opz : g.oz);
  g.tiles_x = (g.ox + TX - 1) / TX;
  g.tiles_y = (g.oy + TY - 1) / TY;
  g.tiles_z = (g.oz + TZ - 1) / TZ;
  g.relu = relu ? 1 : 0;
  require(S <= 65535, "conv_direct: batch above 65535 per call");
  if (S == 0 || fo == 0) return;
  if (direct_tc_supported(f, fo, k, in)) {
    launch_direct_tc(c, in, S, n, w, fo, k, bias, relu, out, g.ipz, g.opz);
    return;
  }
  switch (g.kz) {
    case 1: run_direct<1>(c, in, w, bias, out, g); break;
    case 2: run_direct<2>(c, in, w, bias, out, g); break;
    case 3: run_direct<3>(c, in, w, bias, out, g); break;
    case 4: run_direct<4>(c, in, w, bias, out, g); break;
    case 5: run_direct<5>(c, in, w, bias, out, g); break;
    case 6: run_direct<6>(c, in, w, bias, out, g); break;
    case 7: run_direct<7>(c, in, w, bias, out, g); break;
    case 8: run_direct<8>(c, in, w, bias, out, g); break;
    case 9: run_direct<9>(c, in, w, bias, out, g); break;
    default: run_direct<0>(c, in, w, bias, out, g); break;
  }
}

}  // namespace vxg
