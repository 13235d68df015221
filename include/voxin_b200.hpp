// C++ drop-in for the reference's public interface (proj/include/voxin/*.hpp)
// at T = float, backed by the sm_100a kernels of libvxg.so through the C-ABI of
// include/vxg.h.  A reference caller switches by putting this repo's
// `include/` first on the include path (include/voxin/<name>.hpp forwards here,
// so `#include "voxin/execute.hpp"` keeps working) and linking libvxg.so.
// Names, argument meaning, ownership (input Tensor5 taken by value and
// released, output returned by value) and error behaviour
// (std::invalid_argument via require(), vx::resource_exhausted, vx::ParseError)
// are the reference's.  Calls are synchronous (host tensors staged through
// HBM), which keeps the reference's "externally synchronous" contract.
//
//   reference (proj/include/voxin)        here
//   common.hpp:8-44   vec3, require        same
//   shape.hpp:9-51    Shape5               same
//   tensor.hpp:17-202 Tensor5, ComplexTensor, image_view   same containers
//   memory.hpp:16-104 MemoryTracker, ScopedCharge, MemoryAudit   same
//   network.hpp       ConvSpec, PoolSpec, NetworkSpec     same
//   netspec.hpp       ParseError, parse/format_network_spec -> vxg_net_parse
//   cost.hpp:13-34    PrimitiveKind, ResourceEnv            same
//   cost.cpp:107-122  field_of_view                        -> vxg_net_fov
//   fft.hpp:17-61     RadixProfile, optimal_fft_size       same rule
//   layers.hpp:19-144 ConvLayerParams, LayerContext, LayerResult, DirectVariant
//   layers.hpp:142-192 conv_direct                         -> vxg_conv(DIRECT)
//   layers.hpp:203-371 conv_fft_data_parallel / _staged    -> vxg_conv(FFT)
//   task_conv.hpp:415  conv_fft_task_parallel              -> vxg_conv(FFT)
//   layers.hpp:377-470 max_pool / mpf_pool                 -> vxg_max_pool / vxg_mpf_pool
//   layers.hpp:477-520 recombine_fragments                 -> vxg_recombine
//   planner.hpp:46-171 ShapeChain, LayerPlan, ExecutionPlan, PlanOutcome, SearchBounds,
//                      HostModel, DeviceModel, propagate_shapes, optimize_plan
//   execute.hpp:26-96 NetworkWeights, random_weights, ThroughputReport, ExecutionEnv
//   execute.hpp:388-519 execute_plan, serial_execute, measure_throughput
//                                                           -> vxg_model_forward_ex
//
// What differs from the reference, by design:
//   * compute is fp32 on the GPU: the primitives, random_weights and
//     execute_plan accept T = float only (a static_assert names the rule);
//     containers (Tensor5<double>, ...) stay generic so test oracles compile;
//   * every conv kind runs one of two device algorithms (tiled pruned FFT or
//     direct), every pool kind its device kernel; an ExecutionPlan's theta /
//     divisions / sub-batch describe the reference's host+device split and are
//     validated but not needed: the whole plan runs device-resident;
//   * optimize_plan is the device planner: largest-throughput cubic extent in
//     the bounds whose forward fits the HBM budget (the reference's cost-model
//     search over host/device splits is out of scope).
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <variant>
#include <vector>

#include "vxg.h"

namespace vx {

using i64 = std::int64_t;

// ---- common.hpp ---------------------------------------------------------------------

struct resource_exhausted : std::runtime_error {
  explicit resource_exhausted(const std::string& what) : std::runtime_error(what) {}
};

inline void require(bool cond, const char* what) {
  if (!cond) throw std::invalid_argument(what);
}

struct vec3 {
  i64 x = 1, y = 1, z = 1;
  constexpr i64 elements() const { return x * y * z; }
  constexpr bool operator==(const vec3& o) const { return x == o.x && y == o.y && z == o.z; }
  constexpr bool operator!=(const vec3& o) const { return !(*this == o); }
  constexpr i64 operator[](int a) const { return a == 0 ? x : (a == 1 ? y : z); }
  i64& operator[](int a) { return a == 0 ? x : (a == 1 ? y : z); }
  static constexpr vec3 cube(i64 e) { return {e, e, e}; }
  constexpr bool all_positive() const { return x > 0 && y > 0 && z > 0; }
  constexpr i64 max() const { return x > y ? (x > z ? x : z) : (y > z ? y : z); }
};
inline vec3 operator+(vec3 a, vec3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline vec3 operator-(vec3 a, vec3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline vec3 operator*(vec3 a, vec3 b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
inline std::string to_string(const vec3& v) {
  return std::to_string(v.x) + "x" + std::to_string(v.y) + "x" + std::to_string(v.z);
}

// ---- shape.hpp ------------------------------------------------------------------------

struct Shape5 {
  i64 s = 1, f = 1;
  vec3 n;
  constexpr Shape5() = default;
  constexpr Shape5(i64 s_, i64 f_, vec3 n_) : s(s_), f(f_), n(n_) {}
  constexpr Shape5(i64 s_, i64 f_, i64 x, i64 y, i64 z) : s(s_), f(f_), n{x, y, z} {}
  constexpr bool operator==(const Shape5& o) const { return s == o.s && f == o.f && n == o.n; }
  constexpr bool operator!=(const Shape5& o) const { return !(*this == o); }
  constexpr i64 elements() const { return s * f * n.x * n.y * n.z; }
  constexpr i64 voxels() const { return n.elements(); }
  constexpr i64 stride_z() const { return 1; }
  constexpr i64 stride_y() const { return n.z; }
  constexpr i64 stride_x() const { return n.y * n.z; }
  constexpr i64 stride_f() const { return n.x * n.y * n.z; }
  constexpr i64 stride_s() const { return f * n.x * n.y * n.z; }
  constexpr i64 index(i64 is, i64 jf, i64 ix, i64 iy, i64 iz) const {
    return ((((is * f) + jf) * n.x + ix) * n.y + iy) * n.z + iz;
  }
  void validate() const {
    require(s > 0 && f > 0 && n.all_positive(), "Shape5: all extents must be positive");
    const i64 lim = std::numeric_limits<i64>::max();
    i64 acc = s;
    for (i64 d : {f, n.x, n.y, n.z}) {
      require(acc <= lim / d, "Shape5: element count overflows");
      acc *= d;
    }
  }
};
inline std::string to_string(const Shape5& sh) {
  return "(" + std::to_string(sh.s) + "," + std::to_string(sh.f) + "," + to_string(sh.n) + ")";
}

// ---- tensor.hpp ------------------------------------------------------------------------

template <class T>
class Tensor5 {
 public:
  Tensor5() = default;
  explicit Tensor5(Shape5 shape) : shape_(shape) {
    shape_.validate();
    data_.assign(static_cast<std::size_t>(shape_.elements()), T(0));
  }
  Tensor5(Shape5 shape, std::vector<T> data) : shape_(shape), data_(std::move(data)) {
    shape_.validate();
    require(static_cast<i64>(data_.size()) == shape_.elements(), "Tensor5: data size does not match shape");
  }
  const Shape5& shape() const { return shape_; }
  i64 size() const { return static_cast<i64>(data_.size()); }
  bool empty() const { return data_.empty(); }
  const T* data() const { return data_.data(); }
  T* data() { return data_.data(); }
  const T& at(i64 s, i64 f, i64 x, i64 y, i64 z) const {
    return data_[static_cast<std::size_t>(shape_.index(s, f, x, y, z))];
  }
  T& at(i64 s, i64 f, i64 x, i64 y, i64 z) { return data_[static_cast<std::size_t>(shape_.index(s, f, x, y, z))]; }
  const T* image(i64 s, i64 f) const { return data() + shape_.index(s, f, 0, 0, 0); }
  T* image(i64 s, i64 f) { return data() + shape_.index(s, f, 0, 0, 0); }
  void release() {
    data_.clear();
    data_.shrink_to_fit();
  }

 private:
  Shape5 shape_;
  std::vector<T> data_;
};

template <class T>
struct ConstView3 {
  const T* data = nullptr;
  vec3 n;
  const T& at(i64 x, i64 y, i64 z) const { return data[(x * n.y + y) * n.z + z]; }
};
template <class T>
ConstView3<T> image_view(const Tensor5<T>& t, i64 s, i64 f) {
  return {t.image(s, f), t.shape().n};
}

enum class Axis : unsigned char { batch, feature, x, y, z };

// Frequency-domain container (tensor.hpp:77-152): row-major, last storage axis
// fastest; half_extent = full padded length of the halved axis.
template <class T>
class ComplexTensor {
 public:
  using value_type = std::complex<T>;
  ComplexTensor() = default;
  ComplexTensor(std::vector<i64> dims, std::vector<Axis> layout, i64 half_extent = 0)
      : dims_(std::move(dims)), layout_(std::move(layout)), half_extent_(half_extent) {
    require(!dims_.empty() && dims_.size() <= 5, "ComplexTensor: rank must be 1..5");
    require(dims_.size() == layout_.size(), "ComplexTensor: layout rank mismatch");
    i64 total = 1;
    for (i64 d : dims_) {
      require(d > 0, "ComplexTensor: extents must be positive");
      total *= d;
    }
    data_.assign(static_cast<std::size_t>(total), value_type(0));
  }
  int rank() const { return static_cast<int>(dims_.size()); }
  const std::vector<i64>& dims() const { return dims_; }
  const std::vector<Axis>& layout() const { return layout_; }
  i64 half_extent() const { return half_extent_; }
  void set_half_extent(i64 e) { half_extent_ = e; }
  i64 size() const { return static_cast<i64>(data_.size()); }
  const value_type* data() const { return data_.data(); }
  value_type* data() { return data_.data(); }
  i64 index(const std::array<i64, 5>& idx) const {
    i64 off = 0;
    for (int a = 0; a < rank(); ++a) off = off * dims_[std::size_t(a)] + idx[std::size_t(a)];
    return off;
  }
  const value_type& at(const std::array<i64, 5>& idx) const { return data_[std::size_t(index(idx))]; }
  value_type& at(const std::array<i64, 5>& idx) { return data_[std::size_t(index(idx))]; }
  void release() {
    data_.clear();
    data_.shrink_to_fit();
  }

 private:
  std::vector<i64> dims_;
  std::vector<Axis> layout_;
  i64 half_extent_ = 0;
  std::vector<value_type> data_;
};

// ---- memory.hpp ------------------------------------------------------------------------

class MemoryTracker {
 public:
  MemoryTracker() = default;
  explicit MemoryTracker(i64 cap_scalars) : cap_(cap_scalars) {}
  void charge(i64 scalars) {
    if (scalars <= 0) return;
    std::lock_guard<std::mutex> lk(mu_);
    if (cap_ >= 0 && current_ + scalars > cap_)
      throw resource_exhausted("memory cap exceeded: need " + std::to_string(current_ + scalars) +
                               " scalars, cap " + std::to_string(cap_));
    current_ += scalars;
    if (current_ > peak_) peak_ = current_;
  }
  void release(i64 scalars) {
    if (scalars <= 0) return;
    std::lock_guard<std::mutex> lk(mu_);
    current_ -= scalars;
  }
  i64 current() const {
    std::lock_guard<std::mutex> lk(mu_);
    return current_;
  }
  i64 peak() const {
    std::lock_guard<std::mutex> lk(mu_);
    return peak_;
  }
  i64 cap() const { return cap_; }

 private:
  mutable std::mutex mu_;
  i64 current_ = 0, peak_ = 0, cap_ = -1;
};

class ScopedCharge {
 public:
  ScopedCharge() = default;
  ScopedCharge(MemoryTracker* t, i64 scalars) : t_(t), n_(scalars) {
    if (t_) t_->charge(n_);
  }
  ~ScopedCharge() { reset(); }
  ScopedCharge(const ScopedCharge&) = delete;
  ScopedCharge& operator=(const ScopedCharge&) = delete;
  ScopedCharge(ScopedCharge&& o) noexcept : t_(o.t_), n_(o.n_) { o.t_ = nullptr; }
  void reset() {
    if (t_) t_->release(n_);
    t_ = nullptr;
  }

 private:
  MemoryTracker* t_ = nullptr;
  i64 n_ = 0;
};

struct MemoryAudit {
  double peak = 0;   // real-scalar equivalents: the device allocator's high-water mark of the call
  double model = 0;  // real-scalar equivalents: this design's closed-form working set
};

// ---- errors of the C-ABI -> the reference's exception types -----------------------------

class ParseError : public std::runtime_error {
 public:
  ParseError(i64 line, const std::string& message)
      : std::runtime_error("line " + std::to_string(line) + ": " + message), line_(line) {}
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
      // "line N: message" (netspec.hpp:11-20)
      i64 line = 0;
      std::string rest = msg;
      if (msg.rfind("line ", 0) == 0) {
        const std::size_t colon = msg.find(": ");
        line = std::stoll(msg.substr(5, colon - 5));
        if (colon != std::string::npos) rest = msg.substr(colon + 2);
      }
      throw ParseError(line, rest);
    }
    default: throw std::runtime_error(msg);
  }
}

template <class T>
constexpr void require_fp32() {
  static_assert(std::is_same<T, float>::value,
                "voxin_b200: the B200 primitives compute in fp32 (T = float); the reference's "
                "fp64 instantiations have no device counterpart");
}

// One vxg context per GPU: stream, stream-ordered allocator, HBM budget.
class Device {
 public:
  explicit Device(int device = 0, i64 budget_bytes = 0) {
    vxg_ctx* c = nullptr;
    vxg_throw(vxg_ctx_create(device, budget_bytes, &c));
    ctx_.reset(c);
  }
  vxg_ctx* get() const { return ctx_.get(); }
  i64 budget_bytes() const {
    int64_t cur = 0, peak = 0, bud = 0;
    vxg_throw(vxg_ctx_memory(get(), &cur, &peak, &bud));
    return bud;
  }
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

// ---- network.hpp / netspec.hpp ---------------------------------------------------------------

enum class Activation : unsigned char { identity, relu };
enum class PoolMode : unsigned char { plain, fragments };

struct ConvSpec {
  i64 features_out = 1;
  vec3 kernel;
  Activation act = Activation::identity;
};

struct PoolSpec {
  vec3 window;
  std::optional<PoolMode> forced_mode;
};

using LayerSpec = std::variant<ConvSpec, PoolSpec>;

struct NetworkSpec {
  i64 features_in = 1;
  std::vector<LayerSpec> layers;

  i64 conv_count() const {
    i64 c = 0;
    for (const auto& l : layers) c += std::holds_alternative<ConvSpec>(l) ? 1 : 0;
    return c;
  }
  i64 pool_count() const { return static_cast<i64>(layers.size()) - conv_count(); }
  i64 features_entering(std::size_t at) const {
    i64 f = features_in;
    for (std::size_t l = 0; l < at && l < layers.size(); ++l)
      if (const auto* c = std::get_if<ConvSpec>(&layers[l])) f = c->features_out;
    return f;
  }
  i64 features_out() const { return features_entering(layers.size()); }
  void validate() const {
    require(features_in > 0, "NetworkSpec: features_in must be positive");
    require(!layers.empty(), "NetworkSpec: at least one layer required");
    for (const auto& l : layers) {
      if (const auto* c = std::get_if<ConvSpec>(&l)) {
        require(c->features_out > 0, "NetworkSpec: conv features_out must be positive");
        require(c->kernel.all_positive(), "NetworkSpec: conv kernel extents must be positive");
      } else {
        require(std::get<PoolSpec>(l).window.all_positive(), "NetworkSpec: pool window extents must be positive");
      }
    }
  }
};

// The canonical grammar (netspec.hpp:22-35): one extent for a cube, else three.
inline std::string format_network_spec(const NetworkSpec& net) {
  std::ostringstream out;
  auto ext = [&](const vec3& v) {
    if (v.x == v.y && v.y == v.z)
      out << v.x;
    else
      out << v.x << ' ' << v.y << ' ' << v.z;
  };
  out << "input " << net.features_in << '\n';
  for (const LayerSpec& layer : net.layers) {
    if (const auto* conv = std::get_if<ConvSpec>(&layer)) {
      out << "conv " << conv->features_out << ' ';
      ext(conv->kernel);
      if (conv->act == Activation::relu) out << " relu";
    } else {
      const auto& pool = std::get<PoolSpec>(layer);
      out << "pool ";
      ext(pool.window);
      if (pool.forced_mode) out << (*pool.forced_mode == PoolMode::fragments ? " mpf" : " plain");
    }
    out << '\n';
  }
  return out.str();
}

namespace detail {

struct NetHandle {
  struct Del {
    void operator()(vxg_net* n) const { vxg_net_free(n); }
  };
  std::unique_ptr<vxg_net, Del> p;
  explicit NetHandle(const NetworkSpec& net) {
    vxg_net* n = nullptr;
    vxg_throw(vxg_net_parse(format_network_spec(net).c_str(), &n));
    p.reset(n);
  }
  vxg_net* get() const { return p.get(); }
};

}  // namespace detail

// parse_network_spec (netspec.cpp:54-120): the device library's parser, the
// same diagnostics (ParseError with the 1-based line).
inline NetworkSpec parse_network_spec(const std::string& text) {
  vxg_net* raw = nullptr;
  vxg_throw(vxg_net_parse(text.c_str(), &raw));
  std::unique_ptr<vxg_net, detail::NetHandle::Del> h(raw);
  int64_t info[5];
  vxg_throw(vxg_net_info(raw, info));
  NetworkSpec net;
  net.features_in = info[3];
  for (int64_t l = 0; l < info[0]; ++l) {
    int64_t kind = 0, fo = 0, relu = 0, forced = -1, e[3];
    vxg_throw(vxg_net_layer(raw, l, &kind, e, &fo, &relu, &forced));
    if (kind == 0) {
      net.layers.push_back(ConvSpec{fo, vec3{e[0], e[1], e[2]}, relu ? Activation::relu : Activation::identity});
    } else {
      PoolSpec p{vec3{e[0], e[1], e[2]}, std::nullopt};
      if (forced >= 0) p.forced_mode = forced == 1 ? PoolMode::fragments : PoolMode::plain;
      net.layers.push_back(p);
    }
  }
  return net;
}

// ---- cost.hpp ---------------------------------------------------------------------------------

enum class PrimitiveKind : unsigned char {
  direct_naive,
  direct_temp,
  fft_data_parallel,
  fft_task_parallel,
  fft_staged,
  device_direct_default,
  device_direct_precomp,
  device_fft,
  pool_plain,
  pool_fragments,
};

inline const char* to_string(PrimitiveKind k) {
  switch (k) {
    case PrimitiveKind::direct_naive: return "direct-naive";
    case PrimitiveKind::direct_temp: return "direct-temp";
    case PrimitiveKind::fft_data_parallel: return "fft-data-parallel";
    case PrimitiveKind::fft_task_parallel: return "fft-task-parallel";
    case PrimitiveKind::fft_staged: return "fft-staged";
    case PrimitiveKind::device_direct_default: return "device-direct-default";
    case PrimitiveKind::device_direct_precomp: return "device-direct-precomp";
    case PrimitiveKind::device_fft: return "device-fft";
    case PrimitiveKind::pool_plain: return "pool-plain";
    default: return "pool-fragments";
  }
}
constexpr bool is_pool_kind(PrimitiveKind k) {
  return k == PrimitiveKind::pool_plain || k == PrimitiveKind::pool_fragments;
}
constexpr bool is_device_kind(PrimitiveKind k) {
  return k == PrimitiveKind::device_direct_default || k == PrimitiveKind::device_direct_precomp ||
         k == PrimitiveKind::device_fft;
}
// The device algorithm a conv kind runs on (INTEGRATION.md §1's dispatch table).
inline int device_conv_algo(PrimitiveKind k) {
  switch (k) {
    case PrimitiveKind::direct_naive:
    case PrimitiveKind::direct_temp:
    case PrimitiveKind::device_direct_default:
    case PrimitiveKind::device_direct_precomp: return VXG_CONV_DIRECT;
    case PrimitiveKind::fft_data_parallel:
    case PrimitiveKind::fft_task_parallel:
    case PrimitiveKind::fft_staged:
    case PrimitiveKind::device_fft: return VXG_CONV_FFT;
    default: throw std::invalid_argument("execute: not a convolution primitive");
  }
}

struct ResourceEnv {
  double workers = 1;
  double capacity = std::numeric_limits<double>::infinity();
  double fft_overhead = 0;
};

inline vec3 field_of_view(const NetworkSpec& net) {
  net.validate();
  detail::NetHandle h(net);
  int64_t f[3];
  vxg_throw(vxg_net_fov(h.get(), f));
  return {f[0], f[1], f[2]};
}

// ---- fft.hpp (size rule and workspace policy) ---------------------------------------------------

struct RadixProfile {
  std::vector<int> primes{2, 3, 5, 7, 11, 13};
  std::optional<int> max_11_13_exponent_sum;
  static RadixProfile host_default() { return {{2, 3, 5, 7, 11, 13}, 1}; }
  static RadixProfile device_default() { return {{2, 3, 5, 7}, std::nullopt}; }
  static RadixProfile unrestricted() { return {{2, 3, 5, 7, 11, 13}, std::nullopt}; }
  bool admits(i64 n) const {
    if (n <= 0) return false;
    int big = 0;
    for (int p : primes)
      while (n % p == 0) {
        n /= p;
        if (p == 11 || p == 13) ++big;
      }
    return n == 1 && (!max_11_13_exponent_sum || big <= *max_11_13_exponent_sum);
  }
};

inline i64 optimal_fft_size(i64 n, const RadixProfile& profile) {
  require(n > 0, "optimal_fft_size: n must be positive");
  i64 m = n;
  while (!profile.admits(m)) ++m;
  return m;
}
inline vec3 optimal_fft_sizes(vec3 n, const RadixProfile& profile) {
  return {optimal_fft_size(n.x, profile), optimal_fft_size(n.y, profile), optimal_fft_size(n.z, profile)};
}

// Transform scratch policy (fft.hpp:77-91).  The device transforms keep
// their scratch on chip; the fields are kept for source compatibility.
struct FftWorkspace {
  i64 cap_scalars = i64(8) << 20;
  i64 longest_line = 64;
};

// ---- layers.hpp -------------------------------------------------------------------------------------

template <class T>
struct ConvLayerParams {
  Tensor5<T> kernels;
  std::vector<T> bias;
  Activation act = Activation::identity;

  i64 features_out() const { return kernels.shape().s; }
  i64 features_in() const { return kernels.shape().f; }
  vec3 kernel_extents() const { return kernels.shape().n; }
  void validate(const Shape5& input) const {
    require(kernels.shape().f == input.f, "conv: kernel feature count mismatch");
    require(static_cast<i64>(bias.size()) == kernels.shape().s, "conv: bias count mismatch");
    const vec3 k = kernels.shape().n, n = input.n;
    require(k.x <= n.x && k.y <= n.y && k.z <= n.z, "conv: kernel larger than image");
  }
};

template <class T>
struct LayerResult {
  Tensor5<T> output;
  MemoryAudit audit;
};

enum class DirectVariant : unsigned char { naive, temp_buffer };

// Execution knobs (layers.hpp:57-65).  `workers` and `workspace` have no
// device meaning; `cap_tracker` is charged with the host staging (input +
// output) of each call, so a capped environment still turns over-allocation
// into resource_exhausted; `device` selects the GPU (default: device 0).
template <class T>
struct LayerContext {
  i64 workers = 1;
  RadixProfile profile = RadixProfile::host_default();
  FftWorkspace workspace;
  MemoryTracker* cap_tracker = nullptr;
  Device* device = nullptr;

  Device& gpu() const { return device ? *device : Device::global(); }
};

namespace detail {

template <class T>
LayerResult<T> conv(int algo, Tensor5<T> in, const ConvLayerParams<T>& p, const LayerContext<T>& ctx) {
  require_fp32<T>();
  const Shape5 s = in.shape();
  p.validate(s);
  const Shape5 ks = p.kernels.shape();
  const int64_t n[3] = {s.n.x, s.n.y, s.n.z}, k[3] = {ks.n.x, ks.n.y, ks.n.z};
  Tensor5<T> out(Shape5{s.s, ks.s, s.n - ks.n + vec3{1, 1, 1}});
  ScopedCharge staging(ctx.cap_tracker, in.size() + out.size());
  vxg_audit au{};
  vxg_throw(vxg_conv(ctx.gpu().get(), algo, VXG_MEM_HOST, in.data(), s.s, s.f, n, p.kernels.data(), ks.s, k,
                     p.bias.data(), p.act == Activation::relu, out.data(), &au));
  in.release();
  return {std::move(out), MemoryAudit{au.peak, au.model}};
}

template <class T>
LayerResult<T> pool(bool fragments, Tensor5<T> in, vec3 w, const LayerContext<T>& ctx) {
  require_fp32<T>();
  const Shape5 s = in.shape();
  require(w.all_positive(), fragments ? "mpf_pool: window extents must be positive"
                                      : "max_pool: window extents must be positive");
  const int64_t n[3] = {s.n.x, s.n.y, s.n.z}, p[3] = {w.x, w.y, w.z};
  if (fragments)
    require((s.n.x + 1) % w.x == 0 && (s.n.y + 1) % w.y == 0 && (s.n.z + 1) % w.z == 0,
            "mpf_pool: extent+1 must be divisible by the window");
  else
    require(s.n.x % w.x == 0 && s.n.y % w.y == 0 && s.n.z % w.z == 0,
            "max_pool: extents must be divisible by the window");
  const i64 P = fragments ? w.elements() : 1;
  Tensor5<T> out(Shape5{s.s * P, s.f, {s.n.x / w.x, s.n.y / w.y, s.n.z / w.z}});
  ScopedCharge staging(ctx.cap_tracker, in.size() + out.size());
  vxg_audit au{};
  vxg_throw((fragments ? vxg_mpf_pool : vxg_max_pool)(ctx.gpu().get(), VXG_MEM_HOST, in.data(), s.s, s.f, n, p,
                                                        out.data(), &au));
  in.release();
  return {std::move(out), MemoryAudit{au.peak, au.model}};
}

}  // namespace detail

template <class T>
LayerResult<T> conv_direct(Tensor5<T> in, const ConvLayerParams<T>& p, const LayerContext<T>& ctx,
                           DirectVariant = DirectVariant::naive) {
  return detail::conv(VXG_CONV_DIRECT, std::move(in), p, ctx);
}
template <class T>
LayerResult<T> conv_fft_data_parallel(Tensor5<T> in, const ConvLayerParams<T>& p, const LayerContext<T>& ctx) {
  return detail::conv(VXG_CONV_FFT, std::move(in), p, ctx);
}
template <class T>
LayerResult<T> conv_fft_staged(Tensor5<T> in, const ConvLayerParams<T>& p, const LayerContext<T>& ctx) {
  return detail::conv(VXG_CONV_FFT, std::move(in), p, ctx);
}
template <class T>
LayerResult<T> conv_fft_task_parallel(Tensor5<T> in, const ConvLayerParams<T>& p, const LayerContext<T>& ctx) {
  return detail::conv(VXG_CONV_FFT, std::move(in), p, ctx);
}
template <class T>
LayerResult<T> max_pool(Tensor5<T> in, vec3 p, const LayerContext<T>& ctx) {
  return detail::pool(false, std::move(in), p, ctx);
}
template <class T>
LayerResult<T> mpf_pool(Tensor5<T> in, vec3 p, const LayerContext<T>& ctx) {
  return detail::pool(true, std::move(in), p, ctx);
}

// recombine_fragments (layers.hpp:477-520): no context argument, as in the
// reference; runs on the default device.
template <class T>
Tensor5<T> recombine_fragments(const Tensor5<T>& frags, const std::vector<vec3>& windows, i64 original_batch) {
  require_fp32<T>();
  const Shape5 s = frags.shape();
  std::vector<int64_t> w;
  vec3 stride{1, 1, 1};
  for (const vec3& v : windows) {
    require(v.all_positive(), "recombine_fragments: window extents must be positive");
    w.insert(w.end(), {v.x, v.y, v.z});
    stride = stride * v;
  }
  const int64_t n[3] = {s.n.x, s.n.y, s.n.z};
  require(original_batch > 0 && s.s == original_batch * stride.elements(),
          "recombine_fragments: batch does not match the windows");
  Tensor5<T> out(Shape5{original_batch, s.f, stride * s.n});
  vxg_throw(vxg_recombine(Device::global().get(), VXG_MEM_HOST, frags.data(), s.s, s.f, n,
                          w.empty() ? nullptr : w.data(), static_cast<int64_t>(windows.size()), original_batch,
                          out.data()));
  return out;
}

// ---- planner.hpp ---------------------------------------------------------------------------------------

struct HostModel {
  ResourceEnv env;
  double flop_rate = 5e10;
  double fft_c = 2.5;
  RadixProfile profile = RadixProfile::host_default();
};

struct DeviceModel {
  ResourceEnv env;
  double flop_rate = 1e11;
  double direct_flop_rate = 0;
  double fft_c = 2.5;
  double transfer_rate = 2e9;
  RadixProfile profile = RadixProfile::device_default();
  double direct_rate() const { return direct_flop_rate > 0 ? direct_flop_rate : flop_rate; }
  void validate() const { require(flop_rate > 0 && transfer_rate > 0, "DeviceModel: rates must be positive"); }
};

struct Infeasibility {
  i64 layer = -1;
  std::string rule;
};

struct ShapeChain {
  std::vector<Shape5> shapes;
  std::optional<Infeasibility> violation;
  bool ok() const { return !violation.has_value(); }
};

// propagate_shapes (planner.cpp:536-589) through the device library's shape rules.
inline ShapeChain propagate_shapes(const NetworkSpec& net, const Shape5& input, const std::vector<PoolMode>& pool_modes) {
  net.validate();
  input.validate();
  require(input.f == net.features_in, "propagate_shapes: input features must match the network");
  require(i64(pool_modes.size()) == net.pool_count(), "propagate_shapes: one mode per pooling layer required");
  std::size_t pi = 0;
  for (const auto& l : net.layers)
    if (const auto* p = std::get_if<PoolSpec>(&l)) {
      if (p->forced_mode)
        require(*p->forced_mode == pool_modes[pi], "propagate_shapes: assignment conflicts with a forced pooling mode");
      ++pi;
    }
  detail::NetHandle h(net);
  std::vector<int> modes;
  for (PoolMode m : pool_modes) modes.push_back(m == PoolMode::fragments ? 1 : 0);
  std::vector<int64_t> sh(5 * (net.layers.size() + 1));
  int64_t viol = -1;
  const int64_t e[3] = {input.n.x, input.n.y, input.n.z};
  vxg_throw(vxg_net_propagate(h.get(), input.s, e, modes.empty() ? nullptr : modes.data(), sh.data(), &viol));
  ShapeChain chain;
  const std::size_t count = viol < 0 ? net.layers.size() + 1 : std::size_t(viol) + 1;
  for (std::size_t i = 0; i < count; ++i)
    chain.shapes.push_back(Shape5{sh[5 * i], sh[5 * i + 1], vec3{sh[5 * i + 2], sh[5 * i + 3], sh[5 * i + 4]}});
  if (viol >= 0) {
    const LayerSpec& l = net.layers[std::size_t(viol)];
    std::string rule = "conv: kernel larger than image";
    if (std::holds_alternative<PoolSpec>(l)) {
      std::size_t k = 0;
      for (std::size_t i = 0; i < std::size_t(viol); ++i) k += std::holds_alternative<PoolSpec>(net.layers[i]) ? 1 : 0;
      rule = pool_modes[k] == PoolMode::plain ? "pool: extents must be divisible by the window"
                                              : "pool: extent+1 must be divisible by the window";
    }
    chain.violation = Infeasibility{viol, rule};
  }
  return chain;
}

struct SubDivision {
  i64 s0 = 0, s_n = 0;
  i64 f0 = 0, f_n = 0;
  i64 o0 = 0, o_n = 0;
};

struct LayerPlan {
  PrimitiveKind kind = PrimitiveKind::direct_naive;
  bool on_device = false;
  std::vector<SubDivision> divisions;
  double seconds = 0;
  double transfer_seconds = 0;
  double memory = 0;
};

struct ExecutionPlan {
  Shape5 input;
  std::vector<LayerPlan> layers;
  i64 theta = 0;
  i64 device_sub_batch = 0;
  bool pipelined = false;
  double host_peak = 0;
  double device_peak = 0;
  double seconds = 0;
  double voxels = 0;
  double voxels_per_second = 0;
};

struct PlanOutcome {
  std::optional<ExecutionPlan> plan;
  Infeasibility why;
  bool feasible() const { return plan.has_value(); }
};

struct SearchBounds {
  i64 max_extent = 0;  // 0: as large as the HBM budget allows
  i64 min_extent = 0;
  i64 batch = 1;
  bool anisotropic = false;  // device planner: cubic inputs only
  i64 extent_step = 1;
};

namespace detail {

struct ModelHandle {
  struct Del {
    void operator()(vxg_model* m) const { vxg_model_free(m); }
  };
  std::unique_ptr<vxg_model, Del> p;
  vxg_model* get() const { return p.get(); }
};

inline ModelHandle make_model(Device& d, const NetHandle& net, const float* weights) {
  vxg_model* m = nullptr;
  vxg_throw(vxg_model_create(d.get(), net.get(), weights, VXG_MEM_HOST, &m));
  ModelHandle h;
  h.p.reset(m);
  return h;
}

// Device plan of one cubic extent under fixed pool modes: estimated seconds
// and peak bytes, or nullopt if the shape chain breaks.
struct DevicePlan {
  std::vector<int64_t> info;  // 8 per layer (vxg_model_plan_ex)
  double seconds = 0;
  int64_t bytes = 0;
};

inline std::optional<DevicePlan> device_plan(const ModelHandle& m, const NetworkSpec& net, i64 S, i64 e,
                                             const std::vector<int>& modes) {
  DevicePlan p;
  p.info.resize(8 * net.layers.size());
  const int64_t ext[3] = {e, e, e};
  if (vxg_model_plan_ex(m.get(), S, ext, nullptr, modes.empty() ? nullptr : modes.data(), p.info.data(), &p.bytes) !=
      VXG_OK)
    return std::nullopt;
  for (std::size_t l = 0; l < net.layers.size(); ++l) p.seconds += double(p.info[8 * l + 6]) * 1e-9;
  return p;
}

}  // namespace detail

// optimize_plan: the DEVICE planner behind the reference's signature
// (planner.hpp:154-157).  Pool modes: forced ones kept, fragments preferred
// (the mode the reference's search picks for every bundled net, acceptance C9),
// other combinations tried only when no all-fragment extent exists.  Extents:
// cubic, in [max(fov, min_extent), max_extent] (max_extent 0: up to what fits).
// Score: output voxels / estimated device seconds; ties -> smaller peak, then
// smaller extent (planner.cpp tie-break order).  Feasible: the forward's peak
// fits the device's HBM budget (and host.env.capacity, if finite, holds the
// input plus the output).  Conv kinds are device_direct_default / device_fft as
// the device planner picks them.
inline PlanOutcome optimize_plan(const NetworkSpec& net, const HostModel& host, const SearchBounds& bounds) {
  net.validate();
  require(bounds.batch >= 1, "optimize_plan: batch must be positive");
  Device& dev = Device::global();
  const vec3 fov = field_of_view(net);
  const i64 lo = std::max(fov.max(), bounds.min_extent);
  const i64 hi = bounds.max_extent > 0 ? bounds.max_extent : i64(4096);
  const double budget = double(dev.budget_bytes());
  detail::NetHandle nh(net);
  const detail::ModelHandle mh = detail::make_model(dev, nh, nullptr);
  const i64 npool = net.pool_count();
  std::vector<std::vector<int>> mode_sets;
  {
    std::vector<int> pref;
    for (const auto& l : net.layers)
      if (const auto* p = std::get_if<PoolSpec>(&l)) pref.push_back(p->forced_mode ? (*p->forced_mode == PoolMode::fragments) : 1);
    mode_sets.push_back(pref);
    for (i64 mask = 0; mask < (i64(1) << npool); ++mask) {
      std::vector<int> m(static_cast<std::size_t>(npool), 0);
      for (i64 b = 0; b < npool; ++b) m[std::size_t(b)] = int((mask >> b) & 1);
      if (m != pref) mode_sets.push_back(m);
    }
  }
  const i64 fout = net.features_out();
  std::optional<ExecutionPlan> best;
  for (std::size_t ms = 0; ms < mode_sets.size() && !best; ++ms) {
    const std::vector<int>& modes = mode_sets[ms];
    bool forced_ok = true;
    {
      std::size_t k = 0;
      for (const auto& l : net.layers)
        if (const auto* p = std::get_if<PoolSpec>(&l)) {
          if (p->forced_mode && int(*p->forced_mode == PoolMode::fragments) != modes[k]) forced_ok = false;
          ++k;
        }
    }
    if (!forced_ok) continue;
    bool over_budget_run = false;
    for (i64 e = lo; e <= hi; ++e) {
      const auto dp = detail::device_plan(mh, net, bounds.batch, e, modes);
      if (!dp) continue;
      std::vector<PoolMode> pm;
      for (int m : modes) pm.push_back(m ? PoolMode::fragments : PoolMode::plain);
      const ShapeChain chain = propagate_shapes(net, Shape5{bounds.batch, net.features_in, vec3::cube(e)}, pm);
      if (!chain.ok()) continue;
      vec3 out = chain.shapes.back().n;
      i64 frag = 1;
      for (std::size_t l = 0, k = 0; l < net.layers.size(); ++l)
        if (const auto* p = std::get_if<PoolSpec>(&net.layers[l])) {
          if (modes[k++]) {
            out = out * p->window;
            frag *= p->window.elements();
          }
        }
      (void)frag;
      const double in_s = double(bounds.batch) * double(net.features_in) * double(e * e * e);
      const double out_s = double(bounds.batch) * double(fout) * double(out.elements());
      const bool host_ok = !std::isfinite(host.env.capacity) || in_s + out_s <= host.env.capacity;
      if (double(dp->bytes) > budget || !host_ok) {
        // peaks grow with the extent: stop after a run of infeasible extents past a feasible one
        if (best) over_budget_run = true;
        if (over_budget_run && bounds.max_extent == 0) break;
        continue;
      }
      ExecutionPlan p;
      p.input = Shape5{bounds.batch, net.features_in, vec3::cube(e)};
      for (std::size_t l = 0; l < net.layers.size(); ++l) {
        LayerPlan lp;
        const int64_t* o = dp->info.data() + 8 * l;
        if (o[0] == 0)
          lp.kind = o[1] == VXG_CONV_FFT ? PrimitiveKind::device_fft : PrimitiveKind::device_direct_default;
        else
          lp.kind = o[1] == 1 ? PrimitiveKind::pool_fragments : PrimitiveKind::pool_plain;
        lp.on_device = true;
        lp.seconds = double(o[6]) * 1e-9;
        p.layers.push_back(lp);
      }
      p.theta = 0;
      p.device_sub_batch = bounds.batch;
      p.host_peak = in_s + out_s;
      p.device_peak = double(dp->bytes) / 4.0;
      p.seconds = dp->seconds;
      p.voxels = double(bounds.batch) * double(out.elements());
      p.voxels_per_second = p.seconds > 0 ? p.voxels / p.seconds : 0;
      const bool better = !best || p.voxels_per_second > best->voxels_per_second ||
                          (p.voxels_per_second == best->voxels_per_second && p.device_peak < best->device_peak);
      if (better) best = p;
    }
  }
  PlanOutcome po;
  if (best)
    po.plan = best;
  else
    po.why = Infeasibility{-1, "no admissible input extent fits the bounds and the HBM budget"};
  return po;
}

inline PlanOutcome optimize_plan(const NetworkSpec& net, const HostModel& host, const DeviceModel&,
                                 const SearchBounds& bounds) {
  return optimize_plan(net, host, bounds);
}

// ---- execute.hpp -------------------------------------------------------------------------------------

template <class T>
struct NetworkWeights {
  std::vector<ConvLayerParams<T>> convs;

  void validate(const NetworkSpec& net) const {
    require(static_cast<i64>(convs.size()) == net.conv_count(),
            "NetworkWeights: one parameter set per convolutional layer required");
    i64 f = net.features_in;
    std::size_t c = 0;
    for (const LayerSpec& layer : net.layers) {
      const auto* conv = std::get_if<ConvSpec>(&layer);
      if (!conv) continue;
      const ConvLayerParams<T>& p = convs[c++];
      require(p.features_in() == f && p.features_out() == conv->features_out && p.kernel_extents() == conv->kernel &&
                  p.act == conv->act && static_cast<i64>(p.bias.size()) == conv->features_out,
              "NetworkWeights: parameter shape does not match the layer");
      f = conv->features_out;
    }
  }
  // the flat vxg layout: per conv layer kernels (fo, f, k) then biases (fo)
  std::vector<float> flat() const {
    std::vector<float> w;
    for (const auto& p : convs) {
      w.insert(w.end(), p.kernels.data(), p.kernels.data() + p.kernels.size());
      w.insert(w.end(), p.bias.begin(), p.bias.end());
    }
    return w;
  }
};

// random_weights (execute.hpp:50-73): the device library's bit-identical
// generator (mt19937_64, U(+-sqrt(3/fan-in)) kernels, U(+-0.1) biases).
template <class T>
NetworkWeights<T> random_weights(const NetworkSpec& net, std::uint64_t seed) {
  require_fp32<T>();
  net.validate();
  detail::NetHandle h(net);
  std::vector<float> flat(static_cast<std::size_t>(vxg_net_weight_count(h.get())));
  vxg_throw(vxg_random_weights(h.get(), seed, flat.data()));
  NetworkWeights<T> w;
  i64 f = net.features_in;
  std::size_t off = 0;
  for (const LayerSpec& layer : net.layers) {
    const auto* conv = std::get_if<ConvSpec>(&layer);
    if (!conv) continue;
    ConvLayerParams<T> p;
    p.kernels = Tensor5<T>(Shape5{conv->features_out, f, conv->kernel});
    std::copy(flat.begin() + std::ptrdiff_t(off), flat.begin() + std::ptrdiff_t(off + std::size_t(p.kernels.size())),
              p.kernels.data());
    off += std::size_t(p.kernels.size());
    p.bias.assign(flat.begin() + std::ptrdiff_t(off), flat.begin() + std::ptrdiff_t(off + std::size_t(conv->features_out)));
    off += std::size_t(conv->features_out);
    p.act = conv->act;
    w.convs.push_back(std::move(p));
    f = conv->features_out;
  }
  return w;
}

struct ThroughputReport {
  double voxels = 0;                  // recombined dense output voxels, batch included
  double seconds = 0;                 // wall time of the call (upload, forward, download)
  double voxels_per_second = 0;
  std::vector<double> layer_seconds;  // device time per network layer (CUDA events)
  double transfer_seconds = 0;        // device time outside the layers: H2D/D2H copies + recombination
  double host_peak = 0;               // scalars the host holds: input + output
  double device_peak = 0;             // audited device high-water mark, scalars
};

// Knobs of a real run (execute.hpp:89-96).  host_capacity caps the host
// staging (input + output, scalars); `gpu` selects the device (default 0);
// `tuned` runs the measured-time planner (vxg_model_tune) before the forward.
template <class T>
struct ExecutionEnv {
  i64 workers = 1;
  FftWorkspace workspace{i64(1) << 50, 64};
  RadixProfile host_profile = RadixProfile::host_default();
  std::optional<i64> host_capacity;
  std::optional<DeviceModel> device;
  bool real_transfer_sleep = false;
  Device* gpu = nullptr;
  bool tuned = false;
};

// execute_plan (execute.hpp:388-402): the plan's per-layer kinds decide the
// device algorithm of every conv (direct kinds -> direct kernel, fft kinds ->
// tiled pruned FFT) and plain vs fragment pooling; fragment outputs are
// recombined.  The dense output is the reference's for any feasible plan.
template <class T>
std::pair<Tensor5<T>, ThroughputReport> execute_plan(const ExecutionPlan& plan, const NetworkSpec& net,
                                                     const NetworkWeights<T>& weights, Tensor5<T> input,
                                                     const ExecutionEnv<T>& env) {
  require_fp32<T>();
  const auto start = std::chrono::steady_clock::now();
  require(env.workers >= 1, "execute: at least one worker required");
  net.validate();
  weights.validate(net);
  require(plan.layers.size() == net.layers.size(), "execute: plan does not match the network");
  const i64 L = static_cast<i64>(net.layers.size());
  require(plan.theta >= 0 && plan.theta <= L, "execute: split index out of range");
  std::vector<int> algos, modes;
  std::vector<PoolMode> pm;
  for (std::size_t i = 0; i < net.layers.size(); ++i) {
    const PrimitiveKind k = plan.layers[i].kind;
    if (std::holds_alternative<PoolSpec>(net.layers[i])) {
      require(is_pool_kind(k), "execute: plan assigns a non-pooling primitive to a pool layer");
      modes.push_back(k == PrimitiveKind::pool_fragments ? 1 : 0);
      pm.push_back(k == PrimitiveKind::pool_fragments ? PoolMode::fragments : PoolMode::plain);
    } else {
      require(!is_pool_kind(k), "execute: plan assigns a pooling primitive to a conv layer");
      algos.push_back(device_conv_algo(k));
    }
  }
  const ShapeChain chain = propagate_shapes(net, plan.input, pm);
  require(chain.ok(), "execute: plan input does not propagate through the network");
  require(input.shape() == plan.input, "execute: input does not match the plan");
  // output: fragment pools recombined (execute.hpp:219-226)
  Shape5 fin = chain.shapes.back();
  {
    std::size_t k = 0;
    vec3 stride{1, 1, 1};
    for (const auto& l : net.layers)
      if (const auto* p = std::get_if<PoolSpec>(&l))
        if (modes[k++]) stride = stride * p->window;
    fin = Shape5{plan.input.s, fin.f, stride * fin.n};
  }
  MemoryTracker host(env.host_capacity ? *env.host_capacity : i64(-1));
  ScopedCharge staging(&host, input.size() + fin.elements());
  Tensor5<T> dense(fin);
  Device& dev = env.gpu ? *env.gpu : Device::global();
  detail::NetHandle nh(net);
  const std::vector<float> flat = weights.flat();
  const detail::ModelHandle mh = detail::make_model(dev, nh, flat.data());
  const int64_t e[3] = {plan.input.n.x, plan.input.n.y, plan.input.n.z};
  if (env.tuned) vxg_throw(vxg_model_tune(mh.get(), plan.input.s, e));
  vxg_report rep{};
  vxg_throw(vxg_model_forward_ex(mh.get(), VXG_MEM_HOST, input.data(), plan.input.s, e,
                                 algos.empty() ? nullptr : algos.data(), modes.empty() ? nullptr : modes.data(), 0,
                                 dense.data(), &rep));
  input.release();
  ThroughputReport r;
  r.voxels = double(fin.s) * double(fin.voxels());
  r.layer_seconds.assign(rep.layer_seconds, rep.layer_seconds + rep.layers);
  r.layer_seconds.resize(net.layers.size(), 0.0);
  double lsum = 0;
  for (double s : r.layer_seconds) lsum += s;
  r.transfer_seconds = std::max(0.0, rep.seconds - lsum);
  r.host_peak = double(host.peak());
  r.device_peak = rep.device_peak;
  r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
  r.voxels_per_second = r.voxels / r.seconds;
  return {std::move(dense), r};
}

template <class T>
std::pair<std::vector<Tensor5<T>>, ThroughputReport> serial_execute(const ExecutionPlan& plan, const NetworkSpec& net,
                                                                    const NetworkWeights<T>& weights,
                                                                    std::vector<Tensor5<T>> items,
                                                                    const ExecutionEnv<T>& env) {
  require(!items.empty(), "serial_execute: at least one input required");
  std::vector<Tensor5<T>> outputs;
  ThroughputReport total;
  total.layer_seconds.assign(net.layers.size(), 0.0);
  for (Tensor5<T>& item : items) {
    auto res = execute_plan(plan, net, weights, std::move(item), env);
    outputs.push_back(std::move(res.first));
    const ThroughputReport& rep = res.second;
    total.voxels += rep.voxels;
    total.seconds += rep.seconds;
    total.transfer_seconds += rep.transfer_seconds;
    for (std::size_t i = 0; i < rep.layer_seconds.size(); ++i) total.layer_seconds[i] += rep.layer_seconds[i];
    total.host_peak = std::max(total.host_peak, rep.host_peak);
    total.device_peak = std::max(total.device_peak, rep.device_peak);
  }
  total.voxels_per_second = total.voxels / total.seconds;
  return {std::move(outputs), total};
}

// measure_throughput (execute.hpp:508-519): one warm-up, five timed runs, the
// median-time run reported.
template <class T>
ThroughputReport measure_throughput(const ExecutionPlan& plan, const NetworkSpec& net, const NetworkWeights<T>& weights,
                                    const Tensor5<T>& input, const ExecutionEnv<T>& env) {
  (void)execute_plan(plan, net, weights, Tensor5<T>(input), env);
  std::vector<ThroughputReport> runs;
  for (int i = 0; i < 5; ++i) runs.push_back(execute_plan(plan, net, weights, Tensor5<T>(input), env).second);
  std::sort(runs.begin(), runs.end(),
            [](const ThroughputReport& a, const ThroughputReport& b) { return a.seconds < b.seconds; });
  return runs[2];
}

}  // namespace vx
