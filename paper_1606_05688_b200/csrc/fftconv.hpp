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
  int pz = 0;                // z row pitch (elements, >= nz)
  int vx, vy, vz;            // tile step (= valid outputs per tile)
  int ntx, nty, ntz;         // tiles per axis
  int64_t tiles_per_img;
  int64_t f;                 // channels per batch entry
  int64_t m0;                // first (batch, tile) row of this launch
  int64_t mstride;           // rows of the spectrum buffer (layout stride)
  float2* out;               // [w/lw][mstride][f][lw]
  float scale;
  int kind = VXG_K_TILE_FWD; // instrumentation family (images or kernel spectra)
  int lw = 16;               // frequencies per contiguous chunk (16: FFMA path, 2: tensor cores)
  bool pair = false;         // CTA-pair transform (tile_fwd_pair_kernel) where available
};

struct InvTileArgs {
  const float2* spec;        // [w/16][mstride][fo][16]
  int64_t mstride;
  int64_t fo;
  float* dst;                // (S, fo, on)
  int onx, ony, onz;
  int opz = 0;               // output z row pitch (>= onz)
  int64_t oel;
  int vx, vy, vz;            // valid outputs per tile
  int cx, cy, cz;            // crop begin inside the tile (k - 1)
  int ntx, nty, ntz;
  int64_t tiles_per_img;
  int64_t m0;
  const float* bias;
  int relu;
  int lw = 16;
  bool pair = false;         // CTA-pair transform (tile_inv_pair_kernel)
  int64_t nwp = 0;           // frequencies per (row, map) in the spectrum buffer
  // single input map (f = 1) fused with the contraction: spec holds the input
  // spectra X ([w/16][mstride][1][16]) and the inverse multiplies each line by
  // the kernel spectrum of its output map (wsp, [w/16][w_fo][1][16]) on load
  const float2* wsp = nullptr;
  int64_t w_fo = 0;
  int direct_x = 0;          // one-CTA inverse: x lines loaded from HBM into registers (no staging)
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
  int64_t npairs;            // tensor-core path: frequency pairs
  long long* prof = nullptr; // VXG_TC_PROF: per-CTA role cycle counters
  int dbg = 0;               // VXG_TC_DBG experiment switches (results invalid when set)
  int ypair = 0;             // Y pair-major ([w/2][row][map][2]) instead of line-major
  int quad = 1;              // tensor cores: quad-frequency tiles (k_cgemm_q.cu), else pairs
};

extern const int kTileSizes[];
// VXG_TILE_PAIR=0 disables the CTA-pair forward transform in planned layers
bool tile_pair_enabled();
bool inv_pair_enabled();  // VXG_INV_PAIR=0 disables the CTA-pair inverse
extern const int kNumTileSizes;
// frequencies of a T^3 tile padded to a multiple of the chunk width lw
int64_t tile_nwp(int T, int lw);
void init_twiddles();
void launch_tile_fwd(Ctx* c, int T, const FwdTileArgs& a, int64_t nblocks);
void launch_tile_inv(Ctx* c, int T, const InvTileArgs& a, int64_t nblocks);
void launch_cgemm(Ctx* c, const GemmArgs& a, int64_t nwb);          // FFMA, lw = 16
bool cgemm_tc_supported(int64_t f, int64_t fo);
void launch_cgemm_tc(Ctx* c, const GemmArgs& a, int64_t npairs);    // tcgen05, lw = 2
// pre-split (tf32 hi/lo, UMMA layout) kernel spectra for the tensor-core path
// (quad: the layout k_cgemm_q.cu reads; else k_cgemm_tc.cu's)
int64_t tc_wsplit_bytes(int64_t npairs, int64_t f, int64_t fo, bool quad);
void tc_wsplit(Ctx* c, const float2* raw, void* out, int64_t npairs, int64_t f, int64_t fo, bool quad);
// quad-frequency tiles (k_cgemm_q.cu, the default tensor-core contraction):
// sector-complete epilogue stores, pass-split accumulators
bool tc_quad_enabled();
// quad tiles: tf32 + bf16-correction MMAs (default) or the 3xTF32 split
// (VXG_Q_3TF32=1); the pre-split W layout follows the same switch
bool q_bf16_correction();
int64_t q_wsplit_bytes(int64_t npairs, int64_t f, int64_t fo);
void q_wsplit(Ctx* c, const float2* raw, void* out, int64_t npairs, int64_t f, int64_t fo);
void launch_cgemm_q(Ctx* c, const GemmArgs& a, int64_t npairs);

// Tile-size choice for a layer: minimises the modelled cost of transforms +
// contraction over the supported sizes (or honours T_forced > 0).
struct FftPlan {
  int T = 0;
  V3 v;        // valid outputs per tile per axis
  V3 nt;       // tiles per axis
  int64_t tiles = 0;
  int lw = 16;       // X spectrum chunk width (frequencies per 128-byte line)
  int ylw = 16;      // Y chunk width: 2 = pair-major (tcgen05 epilogue writes whole lines,
                     // the CTA-pair inverse gathers its x lines by TMA)
  bool tc = false;   // tcgen05 3xTF32 contraction (else fp32 FFMA)
  bool quad = true;  // tcgen05 tile shape: 4 frequencies x half the maps (k_cgemm_q.cu) or
                     // 2 frequencies x all maps (k_cgemm_tc.cu); the measured planner picks
  bool pair = false;     // forward tile transform on a CTA pair (T >= 24)
  bool inv_pair = false; // inverse tile transform on a CTA pair (T >= 24)
  bool fused_f1 = false; // f = 1, FFMA: the elementwise contraction happens in the inverse's loads (no Y; one CTA or pair)
  int64_t nwp = 0;   // padded frequencies per (row, channel)
  double cost = 0;
};
FftPlan plan_fft(V3 n, V3 k, int64_t f, int64_t fo, int64_t S, int T_forced = 0);
// explicit variant (parity tests / experiments): tile size T, contraction and
// forward-transform kernels chosen by the caller (tc only where supported)
FftPlan plan_fft_forced(V3 n, V3 k, int64_t f, int64_t fo, int64_t S, int T, bool tc, bool pair);

// Device kernel spectra of one layer for tile size T: [w/lw][fo][f][lw], scaled 1/T^3.
void compute_kernel_spectra(Ctx* c, int T, bool tc, bool quad, const float* w, int64_t fo, int64_t f, V3 k,
                            float2* out);
// bytes of one layer's device kernel spectra in the layout plan.lw selects
int64_t kernel_spectra_bytes(const FftPlan& plan, int64_t f, int64_t fo);

// Conv layer drivers on device pointers.  `wspec` (optional) are cached kernel
// spectra for plan.T; otherwise computed into scratch.  spectra_budget bounds
// the per-chunk spectrum buffers (bytes; <= 0: what the context budget leaves).
// ipz / opz: z row pitch of the input / output activations (0: unpadded).
// conv_fft_device returns the spectrum chunk rows it used.
int64_t conv_fft_device(Ctx* c, const float* in, int64_t S, int64_t f, V3 n, const float* w,
                        int64_t fo, V3 k, const float* bias, bool relu, float* out,
                        const FftPlan& plan, const float2* wspec, int64_t spectra_budget,
                        int64_t ipz = 0, int64_t opz = 0);
void conv_direct_device(Ctx* c, const float* in, int64_t S, int64_t f, V3 n, const float* w,
                        int64_t fo, V3 k, const float* bias, bool relu, float* out,
                        int64_t ipz = 0, int64_t opz = 0);

// rows of spectrum chunk the executor reserves per FFT layer (the chunk grows
// into whatever the budget leaves; VXG_FFT_ROWS overrides)
int64_t fft_reserved_rows();
// peak scratch bytes conv_fft_device needs beyond in/out (one chunk of rows)
int64_t fft_chunk_bytes(const FftPlan& plan, int64_t f, int64_t fo, int64_t rows);

}  // namespace vxg
