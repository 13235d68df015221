// C++ drop-in for the reference's layer-primitive and network-forward
// interface (proj/include/voxin/*.hpp) at T = float, backed by the C-ABI of
// include/vxg.h.  A reference user switches by including this header instead
// of voxin/layers.hpp + voxin/execute.hpp and linking libvxg.so; the names,
// argument meaning, ownership (input Tensor5 taken by value, output returned
// by value) and error behaviour (std::invalid_argument, vx::resource_exhausted,
// vx::ParseError) are the reference's.  Calls are synchronous (host tensors),
// which keeps the reference's "externally synchronous" contract.
//
//   reference                                   here
//   vx::Tensor5<T>          tensor.hpp:17-59     vx::Tensor5<float> (same layout)
//   vx::ConvLayerParams     layers.hpp:19-34     same fields
//   conv_direct             layers.hpp:142-192   -> vxg_conv(VXG_CONV_DIRECT)
//   conv_fft_data_parallel  layers.hpp:203-272   -> vxg_conv(VXG_CONV_FFT)
//   conv_fft_staged         layers.hpp:286-371   -> vxg_conv(VXG_CONV_FFT)
//   conv_fft_task_parallel  task_conv.hpp:415    -> vxg_conv(VXG_CONV_FFT)
//   max_pool / mpf_pool     layers.hpp:377-470   -> vxg_max_pool / vxg_mpf_pool
//   recombine_fragments     layers.hpp:477-520   -> vxg_recombine
//   parse_network_spec      netspec.cpp:54       -> vxg_net_parse
//   field_of_view           cost.cpp:107         -> vxg_net_fov
//   random_weights          execute.hpp:50-73    -> vxg_random_weights
//   execute_plan            execute.hpp:388-402  -> vxg_net_forward (all-MPF plan)
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "vxg.h"

namespace vx {

using i64 = std::int64_t;

struct resource_exhausted : std::runtime_error {
  explicit resource_exhausted(const std::string& w) : std::runtime_error(w) {}
};

class ParseError : public std::runtime_error {
 public:
  ParseError(i64 line, const std::string& m) : std::runtime_error(m), line_(line) {}
  i64 line() const { return line_; }

 private:
  i64 line_;
};

inline void vxg_throw(int status) {
  if (status == VXG_OK) return;
  const std::string msg = vxg_last_error();
  switch (status) {
    case VXG_INVALID: throw std::invalid_argument(msg);
    case VXG_EXHAUSTED: throw resource_exhausted(msg);
    case VXG_PARSE: {
      i64 line = 0;
      if (msg.rfind("line ", 0) == 0) line = std::stoll(msg.substr(5));
      throw ParseError(line, msg);
    }
    default: throw std::runtime_error(msg);
  }
}

struct vec3 {
  i64 x = 1, y = 1, z = 1;
  i64 elements() const { return x * y * z; }
  bool operator==(const vec3& o) const { return x == o.x && y == o.y && z == o.z; }
  static vec3 cube(i64 e) { return {e, e, e}; }
};

struct Shape5 {
  i64 s = 1, f = 1;
  vec3 n;
  i64 elements() const { return s * f * n.elements(); }
  bool operator==(const Shape5& o) const { return s == o.s && f == o.f && n == o.n; }
};

template <class T>
class Tensor5 {
 public:
  Tensor5() = default;
  explicit Tensor5(Shape5 sh) : shape_(sh), data_(static_cast<size_t>(sh.elements()), T(0)) {}
  Tensor5(Shape5 sh, std::vector<T> d) : shape_(sh), data_(std::move(d)) {
    if (static_cast<i64>(data_.size()) != sh.elements())
      throw std::invalid_argument("Tensor5: data size does not match shape");
  }
  const Shape5& shape() const { return shape_; }
  i64 size() const { return static_cast<i64>(data_.size()); }
  T* data() { return data_.data(); }
  const T* data() const { return data_.data(); }
  T* image(i64 s, i64 f) { return data() + (s * shape_.f + f) * shape_.n.elements(); }
  const T* image(i64 s, i64 f) const { return data() + (s * shape_.f + f) * shape_.n.elements(); }
  void release() {
    data_.clear();
    data_.shrink_to_fit();
  }

 private:
  Shape5 shape_;
  std::vector<T> data_;
};

enum class Activation : unsigned char { identity, relu };

template <class T>
struct ConvLayerParams {
  Tensor5<T> kernels;  // (f_out, f_in, k)
  std::vector<T> bias;
  Activation act = Activation::identity;
};

struct MemoryAudit {
  double peak = 0, model = 0;
};

template <class T>
struct LayerResult {
  Tensor5<T> output;
  MemoryAudit audit;
};

// One device context per thread of use (the GPU-side "LayerContext").
class Device {
 public:
  explicit Device(int device = 0, i64 budget_bytes = 0) {
    vxg_ctx* c = nullptr;
    vxg_throw(vxg_ctx_create(device, budget_bytes, &c));
    ctx_.reset(c);
  }
  vxg_ctx* get() const { return ctx_.get(); }
  static Device& global() {
    static Device d(0);
    return d;
  }

 private:
  struct Del {
    void operator()(vxg_ctx* c) const { vxg_ctx_destroy(c); }
  };
  std::unique_ptr<vxg_ctx, Del> ctx_;
};

namespace detail {
inline LayerResult<float> conv(int algo, Tensor5<float> in, const ConvLayerParams<float>& p,
                               Device& d) {
  const Shape5 s = in.shape();
  const Shape5 ks = p.kernels.shape();
  const i64 n[3] = {s.n.x, s.n.y, s.n.z}, k[3] = {ks.n.x, ks.n.y, ks.n.z};
  if (ks.f != s.f) throw std::invalid_argument("conv: kernel feature count mismatch");
  if (static_cast<i64>(p.bias.size()) != ks.s) throw std::invalid_argument("conv: bias count mismatch");
  if (k[0] > n[0] || k[1] > n[1] || k[2] > n[2])
    throw std::invalid_argument("conv: kernel larger than image");  // layers.hpp:32
  Tensor5<float> out(Shape5{s.s, ks.s, {n[0] - k[0] + 1, n[1] - k[1] + 1, n[2] - k[2] + 1}});
  vxg_audit au{};
  vxg_throw(vxg_conv(d.get(), algo, VXG_MEM_HOST, in.data(), s.s, s.f, n, p.kernels.data(), ks.s, k,
                     p.bias.data(), p.act == Activation::relu, out.data(), &au));
  in.release();
  return {std::move(out), MemoryAudit{au.peak, au.model}};
}
}  // namespace detail

inline LayerResult<float> conv_direct(Tensor5<float> in, const ConvLayerParams<float>& p,
                                      Device& d = Device::global()) {
  return detail::conv(VXG_CONV_DIRECT, std::move(in), p, d);
}
inline LayerResult<float> conv_fft_data_parallel(Tensor5<float> in, const ConvLayerParams<float>& p,
                                                 Device& d = Device::global()) {
  return detail::conv(VXG_CONV_FFT, std::move(in), p, d);
}
inline LayerResult<float> conv_fft_staged(Tensor5<float> in, const ConvLayerParams<float>& p,
                                          Device& d = Device::global()) {
  return detail::conv(VXG_CONV_FFT, std::move(in), p, d);
}
inline LayerResult<float> conv_fft_task_parallel(Tensor5<float> in, const ConvLayerParams<float>& p,
                                                 Device& d = Device::global()) {
  return detail::conv(VXG_CONV_FFT, std::move(in), p, d);
}

inline LayerResult<float> pool(bool fragments, Tensor5<float> in, vec3 w, Device& d) {
  const Shape5 s = in.shape();
  const i64 n[3] = {s.n.x, s.n.y, s.n.z}, p[3] = {w.x, w.y, w.z};
  if (w.x <= 0 || w.y <= 0 || w.z <= 0) throw std::invalid_argument("pool: window extents must be positive");
  const i64 P = fragments ? w.elements() : 1;
  Tensor5<float> out(Shape5{s.s * P, s.f, {n[0] / p[0], n[1] / p[1], n[2] / p[2]}});
  vxg_audit au{};
  vxg_throw((fragments ? vxg_mpf_pool : vxg_max_pool)(d.get(), VXG_MEM_HOST, in.data(), s.s, s.f,
                                                        n, p, out.data(), &au));
  in.release();
  return {std::move(out), MemoryAudit{au.peak, au.model}};
}
inline LayerResult<float> max_pool(Tensor5<float> in, vec3 p, Device& d = Device::global()) {
  return pool(false, std::move(in), p, d);
}
inline LayerResult<float> mpf_pool(Tensor5<float> in, vec3 p, Device& d = Device::global()) {
  return pool(true, std::move(in), p, d);
}

inline Tensor5<float> recombine_fragments(const Tensor5<float>& frags,
                                          const std::vector<vec3>& windows, i64 original_batch,
                                          Device& d = Device::global()) {
  const Shape5 s = frags.shape();
  std::vector<i64> w;
  vec3 stride{1, 1, 1};
  for (const vec3& v : windows) {
    w.insert(w.end(), {v.x, v.y, v.z});
    stride = vec3{stride.x * v.x, stride.y * v.y, stride.z * v.z};
  }
  const i64 n[3] = {s.n.x, s.n.y, s.n.z};
  Tensor5<float> out(
      Shape5{original_batch, s.f, {stride.x * s.n.x, stride.y * s.n.y, stride.z * s.n.z}});
  vxg_throw(vxg_recombine(d.get(), VXG_MEM_HOST, frags.data(), s.s, s.f, n,
                          w.empty() ? nullptr : w.data(), static_cast<i64>(windows.size()),
                          original_batch, out.data()));
  return out;
}

// Network description + weights + dense sliding-window forward.
class Network {
 public:
  explicit Network(const std::string& text) {
    vxg_net* n = nullptr;
    vxg_throw(vxg_net_parse(text.c_str(), &n));
    net_.reset(n);
  }
  const vxg_net* get() const { return net_.get(); }
  vec3 field_of_view() const {
    i64 f[3];
    vxg_throw(vxg_net_fov(get(), f));
    return {f[0], f[1], f[2]};
  }
  std::vector<float> random_weights(std::uint64_t seed) const {
    std::vector<float> w(static_cast<size_t>(vxg_net_weight_count(get())));
    vxg_throw(vxg_random_weights(get(), seed, w.data()));
    return w;
  }
  i64 features_out() const {
    i64 info[5];
    vxg_throw(vxg_net_info(get(), info));
    return info[4];
  }

 private:
  struct Del {
    void operator()(vxg_net* n) const { vxg_net_free(n); }
  };
  std::unique_ptr<vxg_net, Del> net_;
};

// execute_plan with an all-fragment plan: (dense output, report)
inline std::pair<Tensor5<float>, vxg_report> execute(const Network& net,
                                                     const std::vector<float>& weights,
                                                     Tensor5<float> input,
                                                     Device& d = Device::global()) {
  const Shape5 s = input.shape();
  const vec3 fov = net.field_of_view();
  const i64 e[3] = {s.n.x, s.n.y, s.n.z};
  Tensor5<float> out(Shape5{s.s, net.features_out(),
                            {s.n.x - fov.x + 1, s.n.y - fov.y + 1, s.n.z - fov.z + 1}});
  vxg_report rep{};
  vxg_throw(vxg_net_forward(d.get(), net.get(), weights.data(), VXG_MEM_HOST, input.data(), s.s, e,
                            nullptr, out.data(), &rep));
  return {std::move(out), rep};
}

}  // namespace vx
