// Drop-in check of include/voxin (the reference's public API at T = float):
// a reference-style C++ caller runs a bundled net file unchanged
// (parse_network_spec -> random_weights<float> -> optimize_plan ->
// execute_plan, proj/include/voxin/execute.hpp:388-402) and exercises the
// reference's error conventions, writing the dense output as raw floats for
// the Python test to compare against the reference's golden vectors.
//   usage: shim_net <net file> <extent> <weight seed> <input seed> <out.bin>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>

#include "voxin/execute.hpp"
#include "voxin/netspec.hpp"
#include "voxin/planner.hpp"

using namespace vx;

int main(int argc, char** argv) {
  if (argc != 6) {
    std::cerr << "usage: shim_net net extent wseed iseed out.bin\n";
    return 2;
  }
  std::ifstream f(argv[1]);
  std::stringstream ss;
  ss << f.rdbuf();
  const i64 e = std::atoll(argv[2]);
  const std::uint64_t wseed = std::strtoull(argv[3], nullptr, 10);
  const std::uint64_t iseed = std::strtoull(argv[4], nullptr, 10);
  try {
    const NetworkSpec net = parse_network_spec(ss.str());
    if (parse_network_spec(format_network_spec(net)).layers.size() != net.layers.size()) return 6;
    const NetworkWeights<float> w = random_weights<float>(net, wseed);
    SearchBounds bounds;
    bounds.min_extent = e;
    bounds.max_extent = e;
    const PlanOutcome po = optimize_plan(net, HostModel{}, bounds);
    if (!po.feasible()) {
      std::cerr << "infeasible: " << po.why.rule << "\n";
      return 7;
    }
    Tensor5<float> x(po.plan->input);
    vxg_fill_random(x.data(), x.size(), iseed);
    ExecutionEnv<float> env;
    auto [dense, rep] = execute_plan(*po.plan, net, w, std::move(x), env);
    std::ofstream o(argv[5], std::ios::binary);
    o.write(reinterpret_cast<const char*>(dense.data()), std::streamsize(sizeof(float) * dense.size()));
    std::cout << "voxels " << rep.voxels << " seconds " << rep.seconds << " layers " << rep.layer_seconds.size()
              << "\n";
    // error behaviour: a malformed net raises vx::ParseError with its line
    try {
      parse_network_spec("input 1\nconv 2 x\n");
      return 3;
    } catch (const ParseError& pe) {
      if (pe.line() != 2) return 4;
    }
    // a kernel larger than the image raises std::invalid_argument
    try {
      ConvLayerParams<float> p;
      p.kernels = Tensor5<float>(Shape5{1, 1, vec3::cube(5)});
      p.bias = {0.f};
      LayerContext<float> ctx;
      conv_direct(Tensor5<float>(Shape5{1, 1, vec3::cube(3)}), p, ctx);
      return 5;
    } catch (const std::invalid_argument&) {
    }
    // a capped tracker turns host over-allocation into resource_exhausted
    try {
      ExecutionEnv<float> tight;
      tight.host_capacity = 100;
      Tensor5<float> x2(po.plan->input);
      execute_plan(*po.plan, net, w, std::move(x2), tight);
      return 8;
    } catch (const resource_exhausted&) {
    }
  } catch (const std::exception& ex) {
    std::cerr << "error: " << ex.what() << "\n";
    return 1;
  }
  return 0;
}
