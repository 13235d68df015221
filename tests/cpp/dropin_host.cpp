// CPU-side drop-in check (no GPU needed): the reference's host-side API at
// T = float -- parse/format, field_of_view, propagate_shapes, random_weights,
// NetworkWeights::validate -- through include/voxin, printing a summary the
// Python test compares with the reference's golden values.
#include <iostream>

#include "voxin/execute.hpp"
#include "voxin/netspec.hpp"
#include "voxin/planner.hpp"

using namespace vx;

int main() {
  NetworkSpec net;
  net.features_in = 1;
  net.layers = {ConvSpec{4, vec3::cube(3), Activation::relu}, PoolSpec{vec3::cube(2), PoolMode::fragments},
                ConvSpec{4, vec3::cube(3), Activation::relu}, PoolSpec{vec3::cube(2), std::nullopt},
                ConvSpec{2, vec3{3, 2, 1}, Activation::identity}};
  std::cout << "fov " << to_string(field_of_view(net)) << "\n";
  std::cout << "format " << format_network_spec(net);
  const NetworkSpec back = parse_network_spec(format_network_spec(net));
  std::cout << "roundtrip " << (format_network_spec(back) == format_network_spec(net)) << "\n";
  const ShapeChain ok = propagate_shapes(net, Shape5{1, 1, vec3::cube(21)},
                                         {PoolMode::fragments, PoolMode::fragments});
  std::cout << "chain " << ok.ok() << " " << to_string(ok.shapes.back()) << "\n";
  const ShapeChain bad = propagate_shapes(net, Shape5{1, 1, vec3::cube(22)}, {PoolMode::fragments, PoolMode::plain});
  std::cout << "violation " << bad.violation->layer << " " << bad.violation->rule << "\n";
  const NetworkWeights<float> w = random_weights<float>(net, 9003);
  w.validate(net);
  std::cout << "w0 " << w.convs[0].kernels.data()[0] << " b0 " << w.convs[0].bias[0] << "\n";
  try {
    propagate_shapes(net, Shape5{1, 1, vec3::cube(21)}, {PoolMode::plain, PoolMode::fragments});
  } catch (const std::invalid_argument& e) {
    std::cout << "forced " << e.what() << "\n";
  }
  NetworkSpec forced = net;
  std::get<PoolSpec>(forced.layers[1]).forced_mode = PoolMode::plain;
  try {
    propagate_shapes(forced, Shape5{1, 1, vec3::cube(21)}, {PoolMode::fragments, PoolMode::fragments});
  } catch (const std::invalid_argument& e) {
    std::cout << "forced " << e.what() << "\n";
  }
  try {
    parse_network_spec("input 1\nconv 4 3\npool 0\n");
  } catch (const ParseError& e) {
    std::cout << "parse " << e.line() << " " << e.what() << "\n";
  }
  return 0;
}
