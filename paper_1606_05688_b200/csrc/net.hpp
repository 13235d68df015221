// Host-side network description, shape rules and synthetic data — the parts
// of the reference's model/planning layer the device forward needs.
//   NetworkSpec / LayerSpec     proj/include/voxin/network.hpp:11-65
//   parse/format                proj/src/netspec.cpp:54-151
//   field_of_view               proj/src/cost.cpp:107-122
//   propagate_shapes            proj/src/planner.cpp:536-589
//   random_weights              proj/include/voxin/execute.hpp:50-73
//   fill_random                 proj/src/cli.cpp:78-84
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"

namespace vxg {

struct Layer {
  int kind = 0;        // 0 conv, 1 pool
  V3 ext;              // kernel or window extents
  i64 fo = 1;          // conv output maps
  bool relu = false;   // conv activation
  int forced = -1;     // pool: -1 auto, 0 plain, 1 fragments
};

struct Net {
  i64 fin = 1;
  std::vector<Layer> layers;

  i64 conv_count() const;
  i64 pool_count() const;
  i64 features_out() const;
  void validate() const;
  i64 weight_count() const;
};

// (s, f, n) per layer boundary
struct Shape {
  i64 s = 1, f = 1;
  V3 n;
};

Net parse_net(const std::string& text);          // throws parse_failure("line N: ...")
std::string format_net(const Net& net);
V3 field_of_view(const Net& net);
// modes: one per pool (0 plain, 1 fragments); empty = all fragments.
// Returns the chain; *violation = offending layer or -1.
std::vector<Shape> propagate_shapes(const Net& net, Shape input, const std::vector<int>& modes,
                                    i64* violation);
void random_weights(const Net& net, uint64_t seed, float* out);
void fill_random(float* out, i64 count, uint64_t seed);

}  // namespace vxg

struct vxg_net {
  vxg::Net net;
};
