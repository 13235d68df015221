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
};

// Per-forward plan: shapes per layer boundary for ONE input entry, resolved
// conv algorithms, pool modes.
struct ForwardPlan {
  std::vector<Shape> shapes;          // per entry (s = fragments produced so far)
  std::vector<LayerChoice> choice;    // per layer (conv layers only meaningful)
  std::vector<int> pool_mode;         // per layer: 1 fragments, 0 plain (pools only)
  std::vector<int64_t> windows;       // fragment windows (network order), flat x3
  int64_t S = 1;
  V3 dense;
  int64_t f_out = 1;
  int64_t alpha = 1;                  // fragments per input entry
};

struct Model {
  Ctx* c = nullptr;
  Net net;
  std::vector<int> conv_index;        // layer -> conv ordinal or -1
  std::vector<DevBuf> kern, bias;     // per conv ordinal
  std::map<std::pair<int, int>, DevBuf> spectra;  // (conv ordinal, T) -> kernel spectra

  Model(Ctx* ctx, const Net& n, const float* weights, bool device_ptr);
  ForwardPlan plan(int64_t S, V3 e, const int* conv_algos) const;
  // bytes the forward needs (inputs + output included) when every FFT layer
  // gets contractions of at least target_rows rows (0: groups of one entry)
  int64_t plan_bytes(const ForwardPlan& p, bool cache_spectra, int64_t target_rows = 0) const;
  // runs the forward on a device input; writes the dense output (device);
  // layer_seconds (optional) gets per-layer device time
  void forward(const ForwardPlan& p, const float* d_in, float* d_dense, bool cache_spectra,
               std::vector<double>* layer_seconds);
  const float2* spectra_for(int ci, const FftPlan& plan, bool cache);
};

}  // namespace vxg

struct vxg_model {
  std::unique_ptr<vxg::Model> m;
};
