// The reference-side binding a voxin maintainer adds to route the reference's
// own executor (PlanRunner, proj/include/voxin/execute.hpp:281-317) onto the
// B200 kernels: for T = float every conv kind and both pool kinds call the
// C-ABI of include/vxg.h; other T keep the reference's host primitives.
// Compiled against the REFERENCE headers (it uses the reference's own vx::
// types), never against this repo's drop-in.  The three one-line hooks that
// call it are shown in INTEGRATION.md §1 and applied at build time by
// oracle/build_refcompat.py (to a scratch copy; the reference stays untouched).
#pragma once

#include <string>
#include <type_traits>
#include <utility>

#include "vxg.h"
#include "voxin/cost.hpp"
#include "voxin/layers.hpp"

namespace vxg_bind {

inline vxg_ctx* context() {
  struct Holder {
    vxg_ctx* c = nullptr;
    Holder() {
      if (vxg_ctx_create(0, 0, &c) != VXG_OK) throw std::runtime_error(vxg_last_error());
    }
    ~Holder() { vxg_ctx_destroy(c); }
  };
  static Holder h;
  return h.c;
}

inline void check(int st) {
  if (st == VXG_OK) return;
  if (st == VXG_INVALID) throw std::invalid_argument(vxg_last_error());
  if (st == VXG_EXHAUSTED) throw vx::resource_exhausted(vxg_last_error());
  throw std::runtime_error(vxg_last_error());
}

// host_conv / device_conv: direct kinds -> the direct kernel, fft kinds -> the
// tiled pruned-FFT convolution
inline vx::Tensor5<float> conv(vx::Tensor5<float> in, const vx::ConvLayerParams<float>& p, vx::PrimitiveKind kind) {
  using K = vx::PrimitiveKind;
  const bool direct = kind == K::direct_naive || kind == K::direct_temp || kind == K::device_direct_default ||
                      kind == K::device_direct_precomp;
  p.validate(in.shape());
  const vx::Shape5 s = in.shape();
  const vx::vec3 k = p.kernel_extents();
  const int64_t n3[3] = {s.n.x, s.n.y, s.n.z}, k3[3] = {k.x, k.y, k.z};
  vx::Tensor5<float> out(vx::Shape5{s.s, p.features_out(), s.n - k + vx::vec3{1, 1, 1}});
  check(vxg_conv(context(), direct ? VXG_CONV_DIRECT : VXG_CONV_FFT, VXG_MEM_HOST, in.data(), s.s, s.f, n3,
                 p.kernels.data(), p.features_out(), k3, p.bias.data(), p.act == vx::Activation::relu, out.data(),
                 nullptr));
  return out;
}

// pool: pool_fragments -> mpf_pool kernel, pool_plain -> max_pool kernel
inline vx::Tensor5<float> pool(vx::Tensor5<float> in, const vx::PoolSpec& spec, vx::PrimitiveKind kind) {
  const bool frag = kind == vx::PrimitiveKind::pool_fragments;
  const vx::Shape5 s = in.shape();
  const vx::vec3 w = spec.window;
  const int64_t n3[3] = {s.n.x, s.n.y, s.n.z}, p3[3] = {w.x, w.y, w.z};
  const int64_t P = frag ? w.elements() : 1;
  vx::Tensor5<float> out(vx::Shape5{s.s * P, s.f, {s.n.x / w.x, s.n.y / w.y, s.n.z / w.z}});
  check((frag ? vxg_mpf_pool : vxg_max_pool)(context(), VXG_MEM_HOST, in.data(), s.s, s.f, n3, p3, out.data(),
                                              nullptr));
  return out;
}

}  // namespace vxg_bind
