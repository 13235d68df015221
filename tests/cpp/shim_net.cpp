// Drop-in check of include/voxin_b200.hpp: a reference-style C++ caller runs
// a bundled net file unchanged (parse -> random_weights -> execute) and a
// few layer primitives, printing the dense output as raw floats on stdout
// for the Python test to compare against the reference's golden vectors.
//   usage: shim_net <net file> <extent> <weight seed> <input seed> <out.bin>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>

#include "voxin_b200.hpp"

int main(int argc, char** argv) {
  if (argc != 6) {
    std::cerr << "usage: shim_net net extent wseed iseed out.bin\n";
    return 2;
  }
  std::ifstream f(argv[1]);
  std::stringstream ss;
  ss << f.rdbuf();
  const long long e = std::atoll(argv[2]);
  const std::uint64_t wseed = std::strtoull(argv[3], nullptr, 10);
  const std::uint64_t iseed = std::strtoull(argv[4], nullptr, 10);
  try {
    vx::Network net(ss.str());
    const auto w = net.random_weights(wseed);
    vx::Tensor5<float> x(vx::Shape5{1, 1, vx::vec3::cube(e)});
    vxg_fill_random(x.data(), x.size(), iseed);
    auto [dense, rep] = vx::execute(net, w, std::move(x));
    std::ofstream o(argv[5], std::ios::binary);
    o.write(reinterpret_cast<const char*>(dense.data()), sizeof(float) * dense.size());
    std::cout << "voxels " << rep.voxels << " seconds " << rep.seconds << "\n";
    // error behaviour: a malformed net raises vx::ParseError with its line
    try {
      vx::Network bad("input 1\nconv 2 x\n");
      return 3;
    } catch (const vx::ParseError& pe) {
      if (pe.line() != 2) return 4;
    }
    // a kernel larger than the image raises std::invalid_argument
    try {
      vx::ConvLayerParams<float> p;
      p.kernels = vx::Tensor5<float>(vx::Shape5{1, 1, vx::vec3::cube(5)});
      p.bias = {0.f};
      vx::conv_direct(vx::Tensor5<float>(vx::Shape5{1, 1, vx::vec3::cube(3)}), p);
      return 5;
    } catch (const std::invalid_argument&) {
    }
  } catch (const std::exception& ex) {
    std::cerr << "error: " << ex.what() << "\n";
    return 1;
  }
  return 0;
}
