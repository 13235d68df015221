// K6 / K7: max-pooling fragments (MPF), plain max pooling and fragment
// recombination.  All HBM-bound data movement: one read of the input and one
// write of the output per element.
//
//   mpf_pool            proj/include/voxin/layers.hpp:424-470
//   max_pool            proj/include/voxin/layers.hpp:377-417
//   recombine_fragments proj/include/voxin/layers.hpp:477-520
//
// Bit-exactness: a window max is taken in the reference's scan order
// (qx, qy, qz lexicographic) with the reference's update rule
// `if (v > m) m = v` starting from the first element, so ties between +0 and
// -0 resolve to the same element.  NaN inputs set the context flag, which the
// host turns into VXG_INVALID like check_no_nan (layers.hpp:111-116).
#include <algorithm>

#include "async.cuh"
#include "common.cuh"

namespace vxg {
namespace {

struct PoolGeom {
  int64_t nx, ny, nz;     // input extents
  int64_t mx, my, mz;     // output (fragment) extents
  int px, py, pz;         // window
  int P;                  // fragments per input entry (1 for plain pooling)
  int64_t f;              // feature maps
  int64_t b0;             // first output batch entry produced
  int64_t nb;             // output batch entries produced
};

// One thread per output voxel, z fastest.  Output batch index b = s*P + off
// with off = ox*py*pz + oy*pz + oz (layers.hpp:440-443); fragments with
// P == 1 reduce to plain block pooling at offset 0.
template <int PX, int PY, int PZ>
__global__ void __launch_bounds__(256) pool_kernel(const float* __restrict__ in,
                                                   float* __restrict__ out, PoolGeom g,
                                                   int* __restrict__ nan_flag) {
  const int px = PX > 0 ? PX : g.px, py = PY > 0 ? PY : g.py, pz = PZ > 0 ? PZ : g.pz;
  const int64_t oel = g.mx * g.my * g.mz;
  const int64_t total = g.nb * g.f * oel;
  const int64_t nel = g.nx * g.ny * g.nz;
  bool saw_nan = false;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t v = t % oel;
    const int64_t bf = t / oel;
    const int64_t fm = bf % g.f;
    const int64_t b = g.b0 + bf / g.f;
    const int64_t s = b / g.P;
    const int off = static_cast<int>(b % g.P);
    const int ox = g.P > 1 ? off / (py * pz) : 0;
    const int oy = g.P > 1 ? (off / pz) % py : 0;
    const int oz = g.P > 1 ? off % pz : 0;
    const int64_t z = v % g.mz, y = (v / g.mz) % g.my, x = v / (g.mz * g.my);
    const float* src = in + (s * g.f + fm) * nel;
    const int64_t x0 = ox + x * px, y0 = oy + y * py, z0 = oz + z * pz;
    float m = __ldg(src + (x0 * g.ny + y0) * g.nz + z0);
    // px/py/pz are compile-time constants in the specialised instantiations
#pragma unroll
    for (int qx = 0; qx < px; ++qx)
#pragma unroll
      for (int qy = 0; qy < py; ++qy) {
        const float* row = src + ((x0 + qx) * g.ny + y0 + qy) * g.nz + z0;
#pragma unroll
        for (int qz = 0; qz < pz; ++qz) {
          const float val = __ldg(row + qz);
          saw_nan |= (val != val);
          m = val > m ? val : m;
        }
      }
    out[t] = m;
  }
  if (saw_nan) *nan_flag = 1;
}

template <int PX, int PY, int PZ>
void run_pool(Ctx* c, const float* in, float* out, const PoolGeom& g) {
  const int64_t total = g.nb * g.f * g.mx * g.my * g.mz;
  if (total == 0) return;
  const unsigned grid = grid_for(total, 256, int64_t(c->num_sms) * 32);
  KScope ks(c, VXG_K_POOL, 0.0, 8.0 * double(total));  // read ~= write (P m^3 ~= n^3)
  pool_kernel<PX, PY, PZ><<<grid, 256, 0, c->stream>>>(in, out, g, c->d_flag);
  c->counted();
  check_launch("pool_kernel");
}

void dispatch_pool(Ctx* c, const float* in, float* out, const PoolGeom& g) {
  if (g.px == 2 && g.py == 2 && g.pz == 2)
    run_pool<2, 2, 2>(c, in, out, g);
  else if (g.px == 1 && g.py == 1 && g.pz == 1)
    run_pool<1, 1, 1>(c, in, out, g);
  else
    run_pool<0, 0, 0>(c, in, out, g);
}

// Fast MPF over whole input entries: the dense p-window max filter
// D[x] = max in[x .. x+p) over x < p*m (per axis), de-interleaved by parity
// into the P fragments (D[o + p*x'] = fragment o at x').  Every input element
// is read from HBM once (neighbour reuse through L1) and every output written
// once.  A thread owns one (y, z) column of D for XT consecutive x and keeps
// the last PX row maxima in registers.  32-bit index math inside a plane.
// Output planes may be a channel slice of a wider tensor (f_tot, c0), which
// the executor uses to pool a conv layer's output channel block by block.
struct MpfGeom {
  int nx, ny, nz;       // input extents
  int mx, my, mz;       // fragment extents
  int px, py, pz, P;
  int dx, dy, dz;       // D extents = p * m
  int f;                // channels of the input planes
  int f_tot, c0;        // output channel count and offset
  int tiles_z, tiles_y, tiles_x;
  int64_t planes;       // S * f
  int ipz, opz;         // z row pitch of input / output planes
  int mx_out, x_out0;   // output fragment x extent and x offset (x-slab pooling; mpf222 only)
};

constexpr int MPF_TZ = 32, MPF_TY = 8, MPF_XT = 16;

template <int PX, int PY, int PZ>
__global__ void __launch_bounds__(256) mpf_full_kernel(const float* __restrict__ in,
                                                       float* __restrict__ out, MpfGeom g,
                                                       int* __restrict__ nan_flag) {
  const int px = PX > 0 ? PX : g.px, py = PY > 0 ? PY : g.py, pz = PZ > 0 ? PZ : g.pz;
  const int tile = blockIdx.x;
  const int tz = tile % g.tiles_z, ty = (tile / g.tiles_z) % g.tiles_y, tx = tile / (g.tiles_z * g.tiles_y);
  const int z = tz * MPF_TZ + threadIdx.x % MPF_TZ;
  const int y = ty * MPF_TY + threadIdx.x / MPF_TZ;
  const int x0 = tx * MPF_XT;
  const int x1 = min(x0 + MPF_XT, g.dx);
  const bool live = z < g.dz && y < g.dy;
  bool saw_nan = false;
  const int64_t nel = int64_t(g.nx) * g.ny * g.ipz;
  const int moel = g.mx * g.my * g.opz;
  const int zo = z / pz, yo = y / py;
  const int offyz = (y % py) * pz + (z % pz);
  for (int64_t plane = blockIdx.y; plane < g.planes; plane += gridDim.y) {
    if (!live) break;
    const int64_t s = plane / g.f;
    const int fm = int(plane % g.f);
    const float* src = in + plane * nel;
    float* dst0 = out + ((s * g.P) * g.f_tot + g.c0 + fm) * int64_t(moel) + int64_t(yo) * g.opz + zo;
    const int64_t fstride = int64_t(g.f_tot) * moel;  // one fragment further
    if (PX == 2 && PY == 2 && PZ == 2 && x1 - x0 == MPF_XT && z + 1 < g.nz && y + 1 < g.ny) {
      // hot path: all 4 * (XT + 1) loads issued before any use
      float v[MPF_XT + 1][4];
#pragma unroll
      for (int r = 0; r <= MPF_XT; ++r) {
        const float* row = src + (int64_t(x0 + r) * g.ny + y) * g.ipz + z;
        v[r][0] = __ldg(row);
        v[r][1] = __ldg(row + 1);
        v[r][2] = __ldg(row + g.ipz);
        v[r][3] = __ldg(row + g.ipz + 1);
      }
      float prev = 0.f;
#pragma unroll
      for (int r = 0; r <= MPF_XT; ++r) {
        float m = v[r][0];
#pragma unroll
        for (int q = 1; q < 4; ++q) {
          saw_nan |= (v[r][q] != v[r][q]);
          m = v[r][q] > m ? v[r][q] : m;
        }
        saw_nan |= (v[r][0] != v[r][0]);
        if (r > 0) {
          const int xd = x0 + r - 1;
          const float d = m > prev ? m : prev;
          const int off = (xd & 1) * 4 + offyz;
          dst0[off * fstride + int64_t(xd >> 1) * g.my * g.opz] = d;
        }
        prev = m;
      }
      continue;
    }
    float r[8];                                       // ring of row maxima (px <= 8)
    for (int x = x0; x < x1 + px - 1; ++x) {
      const float* row = src + (int64_t(x) * g.ny + y) * g.ipz + z;
      float m = __ldg(row);
#pragma unroll
      for (int qy = 0; qy < py; ++qy)
#pragma unroll
        for (int qz = 0; qz < pz; ++qz) {
          const float v = __ldg(row + qy * g.ipz + qz);
          saw_nan |= (v != v);
          m = v > m ? v : m;
        }
      // shift in; emit D[x - px + 1] once px rows are available
      if (PX == 2) {
        r[0] = r[1];
        r[1] = m;
      } else {
        for (int i = 0; i < px - 1; ++i) r[i] = r[i + 1];
        r[px - 1] = m;
      }
      const int xd = x - px + 1;
      if (xd >= x0) {
        float d = r[0];
        for (int i = 1; i < px; ++i) d = r[i] > d ? r[i] : d;
        const int off = (xd % px) * py * pz + offyz;
        dst0[off * fstride + int64_t(xd / px) * g.my * g.opz] = d;
      }
    }
  }
  if (saw_nan) *nan_flag = 1;
}

// p = 2 MPF, HBM-rate version: the CTA stages its input box
// (XT+1) x (TY+1) x (TZ+1) in shared memory with coalesced cp.async (every
// input element crosses the load path once), then each thread walks x down
// one (y, z) column computing the 2x2 row maxima and the 2-row D values from
// shared memory, writing each D value to its fragment.  Same scan order and
// update rule as the reference (first of equal elements wins).
// Each thread owns two adjacent z columns so a warp writes 32 consecutive
// floats (a full 128-byte line) into each of the two z-parity fragments.
constexpr int M2_TZ = 64, M2_TY = 8, M2_XT = 16;
// box rows padded to 68 floats (16-byte multiple): with 16-byte aligned input
// rows (the network forward's padded pitch) a row is 17 16-byte copies
constexpr int M2_BZ = M2_TZ + 4, M2_BY = M2_TY + 1, M2_BX = M2_XT + 1;

__global__ void __launch_bounds__(256) mpf222_kernel(const float* __restrict__ in,
                                                     float* __restrict__ out, MpfGeom g,
                                                     int* __restrict__ nan_flag) {
  __shared__ __align__(16) float box[M2_BX * M2_BY * M2_BZ];
  const int tile = blockIdx.x;
  const int tz = tile % g.tiles_z, ty = (tile / g.tiles_z) % g.tiles_y, tx = tile / (g.tiles_z * g.tiles_y);
  const int z0 = tz * M2_TZ, y0 = ty * M2_TY, x0 = tx * M2_XT;
  const int lz = threadIdx.x % 32, ly = threadIdx.x / 32;
  const int z = z0 + 2 * lz, y = y0 + ly;  // columns z (even) and z + 1
  const int x1 = min(M2_XT, g.dx - x0);
  const bool live = z < g.dz && y < g.dy;    // dz is even: z + 1 < dz too
  const int64_t nel = int64_t(g.nx) * g.ny * g.ipz;
  const int moel = g.mx_out * g.my * g.opz;
  const int64_t fstride = int64_t(g.f_tot) * moel;
  const int offy = (y & 1) * 2;
  const bool vec = (g.ipz & 3) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  bool saw_nan = false;
  for (int64_t plane = blockIdx.y; plane < g.planes; plane += gridDim.y) {
    const float* src = in + plane * nel;
    __syncthreads();  // previous plane's readers are done with the box
    if (vec) {
      // 16-byte copies: thread per (row, chunk); chunks past the row pitch are
      // zero-filled (the padding inside it is never used nor NaN-scanned)
      for (int u = threadIdx.x; u < M2_BX * M2_BY * (M2_BZ / 4); u += 256) {
        const int r = u / (M2_BZ / 4), ch = u % (M2_BZ / 4);
        const int bx = r / M2_BY, by = r % M2_BY;
        const int gx = x0 + bx, gy = y0 + by;
        const bool ok = gx < g.nx && gy < g.ny && z0 + 4 * ch < g.ipz;
        const float* row = src + (int64_t(gx) * g.ny + gy) * g.ipz + z0 + 4 * ch;
        cp_async16(&box[r * M2_BZ + 4 * ch], ok ? row : src, ok);
      }
    } else {
      // warp per box row, lane = z (coalesced 4-byte copies)
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
      for (int r = w; r < M2_BX * M2_BY; r += 8) {
        const int bx = r / M2_BY, by = r % M2_BY;
        const int gx = x0 + bx, gy = y0 + by;
        const bool rok = gx < g.nx && gy < g.ny;
        const float* row = src + (int64_t(gx) * g.ny + gy) * g.ipz + z0;
#pragma unroll
        for (int bz = lane; bz < M2_BZ; bz += 32) {
          const bool ok = rok && z0 + bz < g.nz;
          cp_async4(&box[r * M2_BZ + bz], ok ? row + bz : src, ok);
        }
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // NaN (mpf_pool rejects NaN, layers.hpp:429): checked on the values the
    // window maxima read -- with an odd extent (every admissible MPF input)
    // each input element lies in some window, so the live threads' reads
    // cover the whole image; zero-filled staging outside it holds no NaN
    if (!live) continue;
    const int64_t s = plane / g.f;
    const int fm = int(plane % g.f);
    const int64_t mstep = int64_t(g.my) * g.opz;  // one fragment x row
    // fragment pointers for D row parity (x even / odd) and column parity
    float* q0 = out + ((s * g.P) * g.f_tot + g.c0 + fm) * int64_t(moel) + int64_t(y >> 1) * g.opz +
                (z >> 1) + int64_t((x0 >> 1) + g.x_out0) * mstep;
    float* qe0 = q0 + int64_t(0 + offy) * fstride;
    float* qe1 = q0 + int64_t(1 + offy) * fstride;
    float* qo0 = q0 + int64_t(4 + offy) * fstride;
    float* qo1 = q0 + int64_t(5 + offy) * fstride;
    const float* col = box + ly * M2_BZ + 2 * lz;
    // 2x2 (y, z) maxima of box row xr for columns z and z + 1, in the
    // reference's scan order (first of equal elements wins)
    auto rowmax = [&](int xr, float& m0, float& m1) {
      const float* rw = col + xr * (M2_BY * M2_BZ);
      const float2 a01 = *reinterpret_cast<const float2*>(rw);
      const float2 b01 = *reinterpret_cast<const float2*>(rw + M2_BZ);
      const float a2 = rw[2], b2 = rw[M2_BZ + 2];
      m0 = a01.x;
      m0 = a01.y > m0 ? a01.y : m0;
      m0 = b01.x > m0 ? b01.x : m0;
      m0 = b01.y > m0 ? b01.y : m0;
      m1 = a01.y;
      m1 = a2 > m1 ? a2 : m1;
      m1 = b01.y > m1 ? b01.y : m1;
      m1 = b2 > m1 ? b2 : m1;
      saw_nan |= (a01.x != a01.x) | (a01.y != a01.y) | (b01.x != b01.x) | (b01.y != b01.y) | (a2 != a2) |
                 (b2 != b2);
    };
    float p0, p1;
    rowmax(0, p0, p1);
#pragma unroll 2
    for (int xr = 1; xr <= x1; xr += 2) {
      float m0, m1;
      rowmax(xr, m0, m1);  // D row x0 + xr - 1 (even)
      *qe0 = m0 > p0 ? m0 : p0;
      *qe1 = m1 > p1 ? m1 : p1;
      if (xr + 1 > x1) break;
      float n0, n1;
      rowmax(xr + 1, n0, n1);  // D row x0 + xr (odd)
      *qo0 = n0 > m0 ? n0 : m0;
      *qo1 = n1 > m1 ? n1 : m1;
      p0 = n0;
      p1 = n1;
      qe0 += mstep; qe1 += mstep; qo0 += mstep; qo1 += mstep;
    }
  }
  if (saw_nan) *nan_flag = 1;
}

__global__ void nan_check_kernel(const float* __restrict__ x, int64_t n, int* flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float v = __ldg(x + i);
    bad |= (v != v);
  }
  if (bad) *flag = 1;
}

// Recombination as a gather: one thread per dense voxel (coalesced writes).
// Dense coordinate d = off + x * stride per axis; off's mixed-radix digits
// (cumulative stride before each window, layers.hpp:500-507) give the
// per-window offsets, whose lexicographic indices form the fragment number
// with the FIRST window slowest (layers.hpp:494-504).
struct RecGeom {
  int64_t nx, ny, nz;        // fragment extents
  int64_t fpz;               // fragment z row pitch
  int64_t dx, dy, dz;        // dense extents
  int64_t sx, sy, sz;        // total stride per axis
  int64_t f, alpha, S0;
  int nwin;
  int win[8][3];
  int64_t pre[8][3];         // cumulative stride before window w
  int64_t scale[8];          // fragments per unit of window w's index
};

// The fragment a dense voxel comes from is b(s) + fx(dx) + fy(dy) + fz(dz % sz)
// with each term a sum over the windows (recombine_fragments' index
// decomposition, layers.hpp:493-517).
__device__ __forceinline__ int64_t frag_term(const RecGeom& g, int64_t off, int axis) {
  int64_t b = 0;
  for (int w = 0; w < g.nwin; ++w) {
    const int64_t o = (off / g.pre[w][axis]) % g.win[w][axis];
    const int64_t mul = axis == 0 ? int64_t(g.win[w][1]) * g.win[w][2] : (axis == 1 ? g.win[w][2] : 1);
    b += o * mul * g.scale[w];
  }
  return b;
}

// Persistent over groups of rg dense rows (s, fm, dx, dy).  A dense z row
// interleaves sz fragment rows (dense z = sz * zf + oz); gathering it element
// by element made every warp load touch sz fragment rows hundreds of MB apart
// (~0.5 TB/s).  Here the sz fragment rows of rg dense rows are read whole
// (coalesced) into shared memory in dense order, then the dense rows are
// written whole.
constexpr int REC_SMEM_FLOATS = 8192;  // rg * dz floats (dz <= 8192)
constexpr int REC_MAX_PAIRS = 1024;    // rg * sz fragment rows per group

__global__ void __launch_bounds__(256) recombine_kernel(const float* __restrict__ frag,
                                                        float* __restrict__ dense, RecGeom g, int64_t rows,
                                                        int rg) {
  __shared__ float buf[REC_SMEM_FLOATS];
  __shared__ const float* ptab[REC_MAX_PAIRS];  // (row in group, oz) -> fragment row
  const int64_t nel = g.nx * g.ny * g.fpz;
  const int sz = int(g.sz), fz = int(g.nz), dz = int(g.dz);
  const int64_t fstride = g.f * nel;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int64_t row0 = int64_t(blockIdx.x) * rg; row0 < rows; row0 += int64_t(gridDim.x) * rg) {
    const int nr = int(rows - row0 < rg ? rows - row0 : rg);
    for (int p = threadIdx.x; p < nr * sz; p += blockDim.x) {
      const int r = p / sz, oz = p - r * sz;
      const int64_t row = row0 + r;
      const int64_t dy = row % g.dy;
      const int64_t dx = (row / g.dy) % g.dx;
      const int64_t sf = row / (g.dy * g.dx);
      const int64_t fm = sf % g.f, s = sf / g.f;
      const int64_t b = s * g.alpha + frag_term(g, dx % g.sx, 0) + frag_term(g, dy % g.sy, 1) + frag_term(g, oz, 2);
      ptab[p] = frag + b * fstride + fm * nel + ((dx / g.sx) * g.ny + dy / g.sy) * g.fpz;
    }
    __syncthreads();
    // one warp per fragment row: coalesced reads, scattered into dense z order
    for (int p = warp; p < nr * sz; p += nwarps) {
      const float* src = ptab[p];
      float* d = buf + (p / sz) * dz + (p % sz);
      for (int zf = lane; zf < fz; zf += 32) d[zf * sz] = __ldg(src + zf);
    }
    __syncthreads();
    float* dst = dense + row0 * dz;  // rows are consecutive in the dense output
    for (int u = threadIdx.x; u < nr * dz; u += blockDim.x) dst[u] = buf[u];
    __syncthreads();
  }
}

}  // namespace

void launch_mpf(Ctx* c, const float* in, i64 S, i64 f, V3 n, V3 p, float* out, i64 f_tot,
                i64 c0, i64 ipz, i64 opz, i64 mx_out, i64 x_out0) {
  require(p.x <= 8, "mpf: window above 8 along x");
  MpfGeom g{};
  g.nx = int(n.x); g.ny = int(n.y); g.nz = int(n.z);
  g.mx = int(n.x / p.x); g.my = int(n.y / p.y); g.mz = int(n.z / p.z);
  g.mx_out = int(mx_out > 0 ? mx_out : g.mx);
  g.x_out0 = int(x_out0);
  require((g.mx_out == g.mx && g.x_out0 == 0) || (p.x == 2 && p.y == 2 && p.z == 2),
          "mpf: x-slab pooling is implemented for 2x2x2 windows only");
  require(g.x_out0 + g.mx <= g.mx_out, "mpf: x slab outside the output");
  g.px = int(p.x); g.py = int(p.y); g.pz = int(p.z); g.P = int(p.vol());
  g.dx = g.px * g.mx; g.dy = g.py * g.my; g.dz = g.pz * g.mz;
  g.f = int(f);
  g.f_tot = int(f_tot > 0 ? f_tot : f);
  g.c0 = int(c0);
  g.tiles_z = (g.dz + MPF_TZ - 1) / MPF_TZ;
  g.tiles_y = (g.dy + MPF_TY - 1) / MPF_TY;
  g.tiles_x = (g.dx + MPF_XT - 1) / MPF_XT;
  g.planes = S * f;
  g.ipz = int(ipz > 0 ? ipz : n.z);
  g.opz = int(opz > 0 ? opz : g.mz);
  const int64_t tiles = int64_t(g.tiles_z) * g.tiles_y * g.tiles_x;
  if (tiles == 0 || g.planes == 0) return;
  require(tiles < (int64_t(1) << 31), "mpf: grid too large");
  dim3 grid(unsigned(tiles), unsigned(std::min<int64_t>(g.planes, 65535)));
  KScope ks(c, VXG_K_POOL, 0.0,
            4.0 * double(g.planes) * (double(n.x) * n.y * n.z + double(g.P) * g.mx * g.my * g.mz));
  if (g.px == 2 && g.py == 2 && g.pz == 2) {
    MpfGeom h = g;
    h.tiles_z = (g.dz + M2_TZ - 1) / M2_TZ;
    h.tiles_y = (g.dy + M2_TY - 1) / M2_TY;
    h.tiles_x = (g.dx + M2_XT - 1) / M2_XT;
    const int64_t t2 = int64_t(h.tiles_z) * h.tiles_y * h.tiles_x;
    dim3 grid2(unsigned(t2), unsigned(std::min<int64_t>(g.planes, 65535)));
    mpf222_kernel<<<grid2, 256, 0, c->stream>>>(in, out, h, c->d_flag);
  } else
    mpf_full_kernel<0, 0, 0><<<grid, 256, 0, c->stream>>>(in, out, g, c->d_flag);
  c->counted();
  check_launch("mpf_full_kernel");
}

void launch_maxpool(Ctx* c, const float* in, i64 S, i64 f, V3 n, V3 p, float* out) {
  PoolGeom g{n.x, n.y, n.z, n.x / p.x, n.y / p.y, n.z / p.z, int(p.x), int(p.y), int(p.z), 1,
             f, 0, S};
  dispatch_pool(c, in, out, g);
}

void launch_recombine(Ctx* c, const float* frag, i64 nfrag, i64 b0, i64 f, V3 n,
                      const i64* windows, int nwin, float* dense, i64 S0, i64 fpz) {
  require(nwin <= 8, "recombine: at most 8 fragment windows supported");
  require(b0 == 0, "recombine: partial fragment ranges are not supported");
  RecGeom g{};
  g.nx = n.x; g.ny = n.y; g.nz = n.z;
  g.fpz = fpz > 0 ? fpz : n.z;
  g.f = f; g.S0 = S0; g.nwin = nwin;
  int64_t stride[3] = {1, 1, 1};
  int64_t alpha = 1;
  for (int w = 0; w < nwin; ++w) {
    for (int a = 0; a < 3; ++a) {
      g.win[w][a] = int(windows[3 * w + a]);
      g.pre[w][a] = stride[a];
      stride[a] *= windows[3 * w + a];
    }
    alpha *= windows[3 * w] * windows[3 * w + 1] * windows[3 * w + 2];
  }
  int64_t sc = alpha;
  for (int w = 0; w < nwin; ++w) {
    sc /= windows[3 * w] * windows[3 * w + 1] * windows[3 * w + 2];
    g.scale[w] = sc;
  }
  g.alpha = alpha;
  g.sx = stride[0]; g.sy = stride[1]; g.sz = stride[2];
  g.dx = stride[0] * n.x; g.dy = stride[1] * n.y; g.dz = stride[2] * n.z;
  require(nfrag == S0 * alpha, "recombine_fragments: fragment batch mismatch");
  const int64_t total = S0 * f * g.dx * g.dy * g.dz;
  if (total == 0) return;
  KScope ks(c, VXG_K_RECOMBINE, 0.0, 8.0 * double(total));
  require(g.sz <= 256, "recombine: z stride product above 256");
  require(g.dz <= REC_SMEM_FLOATS, "recombine: dense z extent above 8192");
  const int rg = int(std::max<int64_t>(1, std::min<int64_t>({8, REC_SMEM_FLOATS / g.dz, REC_MAX_PAIRS / g.sz})));
  const int64_t rows = S0 * f * g.dx * g.dy;
  recombine_kernel<<<grid_for(rows, rg, int64_t(c->num_sms) * 8), 256, 0, c->stream>>>(frag, dense, g, rows, rg);
  c->counted();
  check_launch("recombine_kernel");
}

void launch_nan_check(Ctx* c, const float* x, i64 count) {
  if (count == 0) return;
  KScope ks(c, VXG_K_OTHER, 0.0, 4.0 * double(count));
  nan_check_kernel<<<grid_for(count, 256, int64_t(c->num_sms) * 16), 256, 0, c->stream>>>(
      x, count, c->d_flag);
  c->counted();
  check_launch("nan_check_kernel");
}

void clear_flag_async(Ctx* c) { VXG_CUDA_CHECK(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream)); }

bool read_and_clear_flag(Ctx* c) {
  int h = 0;
  VXG_CUDA_CHECK(cudaMemcpyAsync(&h, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  VXG_CUDA_CHECK(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
  VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  return h != 0;
}

}  // namespace vxg
