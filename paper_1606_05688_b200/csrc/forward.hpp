// Device-resident network forward (the B200 counterpart of PlanRunner /
// execute_plan, proj/include/voxin/execute.hpp:123-402).
#pragma once

#include <map>
#include <memory>
#include <utility>
#include <vector>

#include "fftconv.hpp"
#include "net.hpp"

namespace vxg {

struct LayerChoice {
  int algo = VXG_CONV_AUTO;  // resolved to DIRECT or FFT
  FftPlan fft;
  bool measured = false;     // tile size chosen from measured costs (Model::tune)
  double seconds = 0;        // estimated seconds of the layer (measured costs, else the model)
};

// Per-forward plan: shapes per layer boundary for ONE input entry, resolved
// conv algorithms, pool modes.
struct ForwardPlan {
  std::vector<Shape> shapes;          // per entry (s = fragments produced so far)
  std::vector<LayerChoice> choice;    // per layer (conv layers only meaningful)
  std::vector<int> pool_mode;         // per layer: 1 fragments, 0 plain (pools only)
  std::vector<int64_t> windows;       // fragment windows (network order), flat x3
  std::vector<int64_t> pz;            // z row pitch per layer boundary (0: the input, unpadded)
  int64_t S = 1;
  V3 dense;
  int64_t f_out = 1;
  int64_t alpha = 1;                  // fragments per input entry
};

// Measured per-layer costs (Model::tune): seconds per spectrum row of the
// tiled FFT convolution for each tile size, seconds per output voxel of the
// direct convolution; keyed by the layer's (f, fo, k).
// LayerCosts::fft keys: tile size T, | kTunePairTiles for the pair-tile
// tensor-core contraction (k_cgemm_tc.cu) instead of the quad tiles
constexpr int kTuneT = 0xFFFF;
constexpr int kTunePairTiles = 1 << 16;

struct LayerCosts {
  // key -> {fixed seconds per launch, seconds per (batch, tile) row}: fitted
  // from two sample sizes (the fixed part is mostly the kernel-spectrum stream)
  std::map<int, std::pair<double, double>> fft;
  double direct_vox = -1;         // seconds per output voxel (all maps), < 0: not measured
};

struct Model {
  Ctx* c = nullptr;
  Net net;
  std::vector<int> conv_index;        // layer -> conv ordinal or -1
  std::vector<DevBuf> kern, bias;     // per conv ordinal
  std::map<std::pair<int, int>, DevBuf> spectra;  // (conv ordinal, T) -> kernel spectra
  std::map<int, LayerCosts> measured;             // conv ordinal -> measured costs
  double pool_elem = -1;                          // measured MPF seconds per input element
  int64_t arena_slack = 0;  // last forward: arena block bytes it never used (not in its audit)

  bool has_weights = true;  // false: a planning-only model (plan / plan_bytes)

  // weights == nullptr: planning-only model (no device weights)
  Model(Ctx* ctx, const Net& n, const float* weights, bool device_ptr);
  // pool_modes: one per pool layer (0 plain, 1 fragments) or nullptr (the
  // network's forced modes, fragments where the network leaves the choice)
  ForwardPlan plan(int64_t S, V3 e, const int* conv_algos, const int* pool_modes = nullptr) const;
  // bytes the forward needs (inputs + output included) when every FFT layer
  // gets contractions of at least target_rows rows (0: groups of one entry)
  int64_t plan_bytes(const ForwardPlan& p, bool cache_spectra, int64_t target_rows = 0) const;
  // runs the forward on a device input; writes the dense output (device);
  // layer_seconds (optional) gets per-layer device time
  // before_output (optional): an event the stream waits on just before the
  // dense output is written (the streaming API lets the previous patch's
  // download from the same buffer run under this forward)
  void forward(const ForwardPlan& p, const float* d_in, float* d_dense, bool cache_spectra,
               std::vector<double>* layer_seconds, cudaEvent_t before_output = nullptr);
  const float2* spectra_for(int ci, const FftPlan& plan, bool cache);
  // Measured-time planning: times every admissible tile size (and the direct
  // kernel where the model gives it a chance) on sample inputs of each conv
  // layer's real (f, fo, k); plan() then picks per layer by measured cost.
  void tune(int64_t S, V3 e);
};

}  // namespace vxg

struct vxg_model {
  std::unique_ptr<vxg::Model> m;
};
