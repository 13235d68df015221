// Host-side interface of the tiled pruned-FFT convolution (k_fftconv.cu) and
// the layer drivers (conv.cu).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace vxg {

struct FwdTileArgs {
  const float* src;
  int64_t img_stride;        // elements per (s, j) image
  int nx, ny, nz;            // image extents
  int vx, vy, vz;            // tile step (= valid outputs per tile)
  int ntx, nty, ntz;         // tiles per axis
  int64_t tiles_per_img;
  int64_t f;                 // channels per batch entry
  int64_t m0;                // first (batch, tile) row of this launch
  int64_t mstride;           // rows of the spectrum buffer (layout stride)
  float2* out;               // [w/16][mstride][f][16]
  float scale;
  int kind = VXG_K_TILE_FWD; // instrumentation family (images or kernel spectra)
};

struct InvTileArgs {
  const float2* spec;        // [w/16][mstride][fo][16]
  int64_t mstride;
  int64_t fo;
  float* dst;                // (S, fo, on)
  int onx, ony, onz;
  int64_t oel;
  int vx, vy, vz;            // valid outputs per tile
  int cx, cy, cz;            // crop begin inside the tile (k - 1)
  int ntx, nty, ntz;
  int64_t tiles_per_img;
  int64_t m0;
  const float* bias;
  int relu;
};

struct GemmArgs {
  const float2* X;           // [w/16][mstride][f][16]
  const float2* W;           // [w/16][fo][f][16]
  float2* Y;                 // [w/16][mstride][fo][16]
  int64_t M;                 // valid rows
  int64_t mstride;
  int f, fo;
  int mblocks, iblocks;
  int T;                     // tile size (for the algorithmic flop count)
};

extern const int kTileSizes[];
extern const int kNumTileSizes;
int64_t tile_nwb(int T);
void init_twiddles();
void launch_tile_fwd(Ctx* c, int T, const FwdTileArgs& a, int64_t nblocks);
void launch_tile_inv(Ctx* c, int T, const InvTileArgs& a, int64_t nblocks);
void launch_cgemm(Ctx* c, const GemmArgs& a, int64_t nwb);

// Tile-size choice for a layer: minimises the modelled cost of transforms +
// contraction over the supported sizes (or honours T_forced > 0).
struct FftPlan {
  int T = 0;
  V3 v;        // valid outputs per tile per axis
  V3 nt;       // tiles per axis
  int64_t tiles = 0;
  int64_t nwb = 0;
  double cost = 0;
};
FftPlan plan_fft(V3 n, V3 k, int64_t f, int64_t fo, int64_t S, int T_forced = 0);

// Device kernel spectra of one layer for tile size T: [nwb][fo][f][16], scaled 1/T^3.
void compute_kernel_spectra(Ctx* c, int T, const float* w, int64_t fo, int64_t f, V3 k,
                            float2* out);

// Conv layer drivers on device pointers.  `wspec` (optional) are cached kernel
// spectra for plan.T; otherwise computed into scratch.  spectra_budget bounds
// the per-chunk spectrum buffers (bytes; <= 0: what the context budget leaves).
void conv_fft_device(Ctx* c, const float* in, int64_t S, int64_t f, V3 n, const float* w,
                     int64_t fo, V3 k, const float* bias, bool relu, float* out,
                     const FftPlan& plan, const float2* wspec, int64_t spectra_budget);
void conv_direct_device(Ctx* c, const float* in, int64_t S, int64_t f, V3 n, const float* w,
                        int64_t fo, V3 k, const float* bias, bool relu, float* out);

// peak scratch bytes conv_fft_device needs beyond in/out (one chunk of rows)
int64_t fft_chunk_bytes(const FftPlan& plan, int64_t f, int64_t fo, int64_t rows);

}  // namespace vxg
