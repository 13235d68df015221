// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A C-ABI wrapper around the UNMODIFIED reference library (voxin, compiled
// straight from /root/reference/proj by oracle/build_ref.sh into
// oracle/_ref/libvoxref.so).  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py load it, as the checker
// and as the reference CPU arm.  Nothing here is reference source: every
// function just calls the reference's public templates.
//
//   ref_conv            -> conv_direct / conv_fft_data_parallel /
//                          conv_fft_task_parallel / conv_fft_staged
//                          (proj/include/voxin/layers.hpp:142-371,
//                           task_conv.hpp:415-442)
//   ref_max_pool/mpf    -> layers.hpp:377-470
//   ref_recombine       -> layers.hpp:477-520
//   ref_*_fft_*         -> fft.hpp:392-457
//   ref_random_weights  -> execute.hpp:50-73
//   ref_fill_random     -> cli.cpp:78-84 (restated: cli.cpp is not built)
//   ref_net_forward     -> execute.hpp:388-402 (host-only plan, theta = L)
//   ref_net_sample      -> the reference primitives timed layer by layer on a
//                          fragment-sampled chain (kept for experiments)
//   ref_stepper_*       -> execute_plan's host-only path (run_prefix +
//                          recombine, execute.hpp:147-164, 219-226, 388-402)
//                          executed one layer per call, with the plan of the
//                          reference's own optimize_plan (planner.cpp:648-686)
//                          or a forced conv kind: bench.py's reference arm and
//                          cpu_baseline (a bench step = one layer of a forward)

#include <chrono>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "voxin/cost.hpp"
#include "voxin/execute.hpp"
#include "voxin/fft.hpp"
#include "voxin/layers.hpp"
#include "voxin/netspec.hpp"
#include "voxin/planner.hpp"
#include "voxin/task_conv.hpp"

using namespace vx;

namespace {

thread_local std::string g_err;
int g_workers = 1;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const resource_exhausted& e) {
    g_err = e.what();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

vec3 v3(const int64_t* a) { return vec3{a[0], a[1], a[2]}; }

template <class T>
Tensor5<T> tensor_from(const void* p, Shape5 sh) {
  Tensor5<T> t(sh);
  std::memcpy(t.data(), p, sizeof(T) * static_cast<size_t>(t.size()));
  return t;
}

template <class T>
void tensor_to(const Tensor5<T>& t, void* p) {
  std::memcpy(p, t.data(), sizeof(T) * static_cast<size_t>(t.size()));
}

template <class T>
LayerContext<T> ctx_of() {
  LayerContext<T> ctx;
  ctx.workers = g_workers;
  ctx.workspace = FftWorkspace{i64(1) << 50, 64};  // as ExecutionEnv (execute.hpp:93)
  return ctx;
}

template <class T>
ConvLayerParams<T> params_of(const void* w, int64_t fo, int64_t f, vec3 k, const void* bias,
                             int relu) {
  ConvLayerParams<T> p;
  p.kernels = tensor_from<T>(w, Shape5{fo, f, k});
  p.bias.assign(static_cast<const T*>(bias), static_cast<const T*>(bias) + fo);
  p.act = relu ? Activation::relu : Activation::identity;
  return p;
}

template <class T>
Tensor5<T> run_conv(int kind, Tensor5<T> in, const ConvLayerParams<T>& p) {
  auto ctx = ctx_of<T>();
  switch (kind) {
    case 0: return conv_direct(std::move(in), p, ctx, DirectVariant::naive).output;
    case 1: return conv_direct(std::move(in), p, ctx, DirectVariant::temp_buffer).output;
    case 2: return conv_fft_data_parallel(std::move(in), p, ctx).output;
    case 3: return conv_fft_task_parallel(std::move(in), p, ctx).output;
    case 4: return conv_fft_staged(std::move(in), p, ctx).output;
    default: throw std::invalid_argument("ref_conv: unknown kind");
  }
}

PrimitiveKind kind_enum(int kind) {
  switch (kind) {
    case 0: return PrimitiveKind::direct_naive;
    case 1: return PrimitiveKind::direct_temp;
    case 2: return PrimitiveKind::fft_data_parallel;
    case 3: return PrimitiveKind::fft_task_parallel;
    case 4: return PrimitiveKind::fft_staged;
    default: throw std::invalid_argument("unknown conv kind");
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_set_workers(int w) {
  g_workers = w > 0 ? w : static_cast<int>(std::thread::hardware_concurrency());
  return g_workers;
}

int ref_conv(int kind, int prec, const void* in, int64_t S, int64_t f, const int64_t* n,
             const void* w, int64_t fo, const int64_t* k, const void* bias, int relu, void* out) {
  return guard([&] {
    if (prec == 64) {
      auto p = params_of<double>(w, fo, f, v3(k), bias, relu);
      tensor_to(run_conv<double>(kind, tensor_from<double>(in, Shape5{S, f, v3(n)}), p), out);
    } else {
      auto p = params_of<float>(w, fo, f, v3(k), bias, relu);
      tensor_to(run_conv<float>(kind, tensor_from<float>(in, Shape5{S, f, v3(n)}), p), out);
    }
  });
}

int ref_pool(int fragments, int prec, const void* in, int64_t S, int64_t f, const int64_t* n,
             const int64_t* p, void* out) {
  return guard([&] {
    if (prec == 64) {
      auto ctx = ctx_of<double>();
      auto t = tensor_from<double>(in, Shape5{S, f, v3(n)});
      tensor_to(fragments ? mpf_pool(std::move(t), v3(p), ctx).output
                          : max_pool(std::move(t), v3(p), ctx).output,
                out);
    } else {
      auto ctx = ctx_of<float>();
      auto t = tensor_from<float>(in, Shape5{S, f, v3(n)});
      tensor_to(fragments ? mpf_pool(std::move(t), v3(p), ctx).output
                          : max_pool(std::move(t), v3(p), ctx).output,
                out);
    }
  });
}

int ref_recombine(int prec, const void* frag, int64_t S, int64_t f, const int64_t* n,
                  const int64_t* windows, int64_t nwin, int64_t original_batch, void* out) {
  return guard([&] {
    std::vector<vec3> win;
    for (int64_t i = 0; i < nwin; ++i) win.push_back(v3(windows + 3 * i));
    if (prec == 64)
      tensor_to(recombine_fragments(tensor_from<double>(frag, Shape5{S, f, v3(n)}), win,
                                    original_batch),
                out);
    else
      tensor_to(recombine_fragments(tensor_from<float>(frag, Shape5{S, f, v3(n)}), win,
                                    original_batch),
                out);
  });
}

// nested pruned forward: out is (floor(px/2)+1, py, pz) complex, interleaved
int ref_pruned_fwd(int prec, const void* img, const int64_t* n, const int64_t* pad, void* out) {
  return guard([&] {
    if (prec == 64) {
      auto t = tensor_from<double>(img, Shape5{1, 1, v3(n)});
      auto s = pruned_fft_forward(image_view(t, 0, 0), v3(pad));
      std::memcpy(out, s.data(), sizeof(double) * 2 * static_cast<size_t>(s.size()));
    } else {
      auto t = tensor_from<float>(img, Shape5{1, 1, v3(n)});
      auto s = pruned_fft_forward(image_view(t, 0, 0), v3(pad));
      std::memcpy(out, s.data(), sizeof(float) * 2 * static_cast<size_t>(s.size()));
    }
  });
}

}  // extern "C"
template <class T>
void pruned_inv_t(const void* spec, const int64_t* pad, const int64_t* crop, void* out) {
  const vec3 p = v3(pad);
  ComplexTensor<T> s({p.x / 2 + 1, p.y, p.z}, {Axis::x, Axis::y, Axis::z}, p.x);
  std::memcpy(s.data(), spec, sizeof(T) * 2 * static_cast<size_t>(s.size()));
  tensor_to(pruned_fft_inverse(std::move(s), v3(crop)), out);
}

extern "C" {
int ref_pruned_inv(int prec, const void* spec, const int64_t* pad, const int64_t* crop, void* out) {
  return guard([&] {
    if (prec == 64)
      pruned_inv_t<double>(spec, pad, crop, out);
    else
      pruned_inv_t<float>(spec, pad, crop, out);
  });
}

// batched forward: out is (b, floor(pz/2)+1, py, px) complex, interleaved
int ref_batched_fwd(int prec, const void* imgs, int64_t b, const int64_t* n, const int64_t* pad,
                    void* out) {
  return guard([&] {
    FftWorkspace ws{i64(1) << 50, 64};
    if (prec == 64) {
      auto t = tensor_from<double>(imgs, Shape5{b, 1, v3(n)});
      auto s = batched_fft_forward(t, v3(pad), ws);
      std::memcpy(out, s.data(), sizeof(double) * 2 * static_cast<size_t>(s.size()));
    } else {
      auto t = tensor_from<float>(imgs, Shape5{b, 1, v3(n)});
      auto s = batched_fft_forward(t, v3(pad), ws);
      std::memcpy(out, s.data(), sizeof(float) * 2 * static_cast<size_t>(s.size()));
    }
  });
}

}  // extern "C"
template <class T>
void batched_inv_t(const void* spec, int64_t b, const int64_t* pad, const int64_t* crop, void* out) {
  const vec3 p = v3(pad);
  ComplexTensor<T> s({b, p.z / 2 + 1, p.y, p.x}, {Axis::batch, Axis::z, Axis::y, Axis::x}, p.z);
  std::memcpy(s.data(), spec, sizeof(T) * 2 * static_cast<size_t>(s.size()));
  FftWorkspace ws{i64(1) << 50, 64};
  tensor_to(batched_fft_inverse(std::move(s), v3(crop), ws), out);
}

extern "C" {
int ref_batched_inv(int prec, const void* spec, int64_t b, const int64_t* pad, const int64_t* crop,
                    void* out) {
  return guard([&] {
    if (prec == 64)
      batched_inv_t<double>(spec, b, pad, crop, out);
    else
      batched_inv_t<float>(spec, b, pad, crop, out);
  });
}

int64_t ref_optimal_fft_size(int64_t n, int profile) {
  int64_t r = -1;
  guard([&] {
    const RadixProfile p = profile == 0   ? RadixProfile::host_default()
                           : profile == 1 ? RadixProfile::device_default()
                                          : RadixProfile::unrestricted();
    r = optimal_fft_size(n, p);
  });
  return r;
}

int ref_fov(const char* net_text, int64_t* fov) {
  return guard([&] {
    const vec3 v = field_of_view(parse_network_spec(net_text));
    fov[0] = v.x;
    fov[1] = v.y;
    fov[2] = v.z;
  });
}

// Shape chain under the given pool modes (0 plain, 1 fragments).  Writes
// (layers+1) x 5 int64 (s, f, x, y, z); *violation = offending layer or -1.
int ref_propagate(const char* net_text, int64_t S, const int64_t* e, const int* modes,
                  int64_t* shapes, int64_t* violation) {
  return guard([&] {
    const NetworkSpec net = parse_network_spec(net_text);
    std::vector<PoolMode> pm;
    for (i64 i = 0; i < net.pool_count(); ++i)
      pm.push_back(modes[i] ? PoolMode::fragments : PoolMode::plain);
    const ShapeChain ch = propagate_shapes(net, Shape5{S, net.features_in, v3(e)}, pm);
    for (size_t i = 0; i < ch.shapes.size(); ++i) {
      const Shape5& s = ch.shapes[i];
      const int64_t row[5] = {s.s, s.f, s.n.x, s.n.y, s.n.z};
      std::memcpy(shapes + 5 * i, row, sizeof(row));
    }
    *violation = ch.ok() ? -1 : ch.violation->layer;
  });
}

// Flat weights: per conv layer in order, kernels (fo, f, k) then biases (fo).
int ref_random_weights(const char* net_text, uint64_t seed, int prec, void* out) {
  return guard([&] {
    const NetworkSpec net = parse_network_spec(net_text);
    size_t off = 0;
    if (prec == 64) {
      auto w = random_weights<double>(net, seed);
      double* o = static_cast<double*>(out);
      for (auto& c : w.convs) {
        std::memcpy(o + off, c.kernels.data(), sizeof(double) * c.kernels.size());
        off += static_cast<size_t>(c.kernels.size());
        std::memcpy(o + off, c.bias.data(), sizeof(double) * c.bias.size());
        off += c.bias.size();
      }
    } else {
      auto w = random_weights<float>(net, seed);
      float* o = static_cast<float*>(out);
      for (auto& c : w.convs) {
        std::memcpy(o + off, c.kernels.data(), sizeof(float) * c.kernels.size());
        off += static_cast<size_t>(c.kernels.size());
        std::memcpy(o + off, c.bias.data(), sizeof(float) * c.bias.size());
        off += c.bias.size();
      }
    }
  });
}

// the bench input generator of cli.cpp:78-84 (mt19937_64, U(-1,1) in double)
int ref_fill_random(int prec, void* out, int64_t count, uint64_t seed) {
  return guard([&] {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> d(-1.0, 1.0);
    if (prec == 64) {
      double* p = static_cast<double*>(out);
      for (int64_t i = 0; i < count; ++i) p[i] = d(rng);
    } else {
      float* p = static_cast<float*>(out);
      for (int64_t i = 0; i < count; ++i) p[i] = static_cast<float>(d(rng));
    }
  });
}

}  // extern "C"
namespace {

ExecutionPlan host_plan(const NetworkSpec& net, Shape5 input, int conv_kind, int mpf) {
  ExecutionPlan plan;
  plan.input = input;
  for (const auto& l : net.layers) {
    LayerPlan lp;
    if (std::holds_alternative<ConvSpec>(l))
      lp.kind = kind_enum(conv_kind);
    else
      lp.kind = mpf ? PrimitiveKind::pool_fragments : PrimitiveKind::pool_plain;
    plan.layers.push_back(lp);
  }
  plan.theta = static_cast<i64>(net.layers.size());
  plan.device_sub_batch = 0;
  return plan;
}

template <class T>
void net_forward_t(const NetworkSpec& net, uint64_t wseed, const void* input, int64_t S,
                   vec3 e, int conv_kind, int mpf, void* out, double* seconds) {
  const auto w = random_weights<T>(net, wseed);
  const ExecutionPlan plan = host_plan(net, Shape5{S, net.features_in, e}, conv_kind, mpf);
  ExecutionEnv<T> env;
  env.workers = g_workers;
  auto [dense, rep] =
      execute_plan(plan, net, w, tensor_from<T>(input, Shape5{S, net.features_in, e}), env);
  tensor_to(dense, out);
  if (seconds) *seconds = rep.seconds;
}

}  // namespace

extern "C" {
// Full network forward through the reference's execute_plan on a host-only
// plan (every conv = conv_kind, every pool MPF when mpf != 0).  Weights are
// random_weights(net, wseed).  out receives the recombined dense output.
int ref_net_forward(const char* net_text, int prec, uint64_t wseed, const void* input, int64_t S,
                    const int64_t* e, int conv_kind, int mpf, void* out, double* seconds) {
  return guard([&] {
    const NetworkSpec net = parse_network_spec(net_text);
    if (prec == 64)
      net_forward_t<double>(net, wseed, input, S, v3(e), conv_kind, mpf, out, seconds);
    else
      net_forward_t<float>(net, wseed, input, S, v3(e), conv_kind, mpf, out, seconds);
  });
}

// CPU-baseline sampler.  Runs the reference's own fp32 primitives layer by
// layer on cubic input extent e (all pools MPF, convs = conv_kind), but after
// every MPF keeps only the first `keep` fragments (0: all) and charges the
// following layers' measured time times (produced / kept).  Returns the
// extrapolated seconds for the full forward; *sample_seconds is the wall time
// actually spent; *dense_voxels the recombined output voxel count.
int ref_net_sample(const char* net_text, int64_t e, uint64_t wseed, uint64_t iseed, int conv_kind,
                   int64_t keep, double* extrapolated, double* sample_seconds,
                   double* dense_voxels) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    const NetworkSpec net = parse_network_spec(net_text);
    const auto w = random_weights<float>(net, wseed);
    Tensor5<float> x(Shape5{1, net.features_in, vec3::cube(e)});
    {
      std::mt19937_64 rng(iseed);
      std::uniform_real_distribution<double> d(-1.0, 1.0);
      for (i64 i = 0; i < x.size(); ++i) x.data()[i] = static_cast<float>(d(rng));
    }
    double mult = 1.0, total = 0.0, spent = 0.0;
    size_t ci = 0;
    auto ctx = ctx_of<float>();
    for (const auto& l : net.layers) {
      const auto t0 = clk::now();
      if (std::holds_alternative<ConvSpec>(l)) {
        // conv_kind < 0: the reference's fastest measured host primitive per
        // layer -- direct for single-input-map layers, task-parallel FFT else
        const int kind = conv_kind >= 0 ? conv_kind : (x.shape().f == 1 ? 0 : 3);
        x = run_conv<float>(kind, std::move(x), w.convs[ci++]);
      } else {
        const vec3 p = std::get<PoolSpec>(l).window;
        x = mpf_pool(std::move(x), p, ctx).output;
        const i64 have = x.shape().s;
        // sample only at the FIRST pool: later layers keep running batched,
        // so per-call overheads are charged as in the full run
        const i64 k = (keep > 0 && mult == 1.0) ? std::min<i64>(keep, have) : have;
        const double dt0 = std::chrono::duration<double>(clk::now() - t0).count();
        total += dt0 * mult;
        spent += dt0;
        if (k < have) {
          Tensor5<float> y(Shape5{k, x.shape().f, x.shape().n});
          std::memcpy(y.data(), x.data(), sizeof(float) * static_cast<size_t>(y.size()));
          mult *= static_cast<double>(have) / static_cast<double>(k);
          x = std::move(y);
        }
        continue;
      }
      const double dt = std::chrono::duration<double>(clk::now() - t0).count();
      total += dt * mult;
      spent += dt;
    }
    const vec3 fov = field_of_view(net);
    const double d = static_cast<double>(e - fov.x + 1);
    *extrapolated = total;
    *sample_seconds = spent;
    *dense_voxels = d * d * d;
  });
}

// Planner entry (for host-logic parity): the reference's optimize_plan on a
// host model, returning the chosen cubic extent and per-layer kinds.
int ref_optimize_plan(const char* net_text, int64_t min_extent, int64_t max_extent,
                      int64_t* extent, int* kinds) {
  return guard([&] {
    const NetworkSpec net = parse_network_spec(net_text);
    SearchBounds b;
    b.min_extent = min_extent;
    b.max_extent = max_extent;
    const PlanOutcome po = optimize_plan(net, HostModel{}, b);
    require(po.feasible(), "no feasible plan");
    *extent = po.plan->input.n.x;
    for (size_t i = 0; i < po.plan->layers.size(); ++i)
      kinds[i] = static_cast<int>(po.plan->layers[i].kind);
  });
}


}  // extern "C"

namespace {

// One forward of execute_plan's host-only path (theta = L), a layer per step.
struct Stepper {
  NetworkSpec net;
  NetworkWeights<float> w;
  ExecutionPlan plan;
  Tensor5<float> input, cur;
  std::vector<i64> conv_at;
  std::vector<vec3> windows;  // fragment windows in network order
  size_t li = 0;
  bool need_input = false;  // a forward completed: the next step starts from the input
};

LayerContext<float> host_ctx() {
  // PlanRunner::host_ctx (execute.hpp:247-255) with ExecutionEnv defaults
  LayerContext<float> ctx;
  ctx.workers = g_workers;
  ctx.workspace = FftWorkspace{i64(1) << 50, 64};
  ctx.profile = RadixProfile::host_default();
  return ctx;
}

}  // namespace

extern "C" {

// plan_mode 0: the reference planner's own plan (optimize_plan on a HostModel
// with workers = the worker count, bounds [e, e]); 1: every conv = conv_kind,
// every pool MPF.  kinds (optional, one per layer) receives the plan's
// PrimitiveKind values.
int ref_stepper_create(const char* net_text, int64_t e, uint64_t wseed, uint64_t iseed, int plan_mode,
                       int conv_kind, void** handle, int* kinds) {
  return guard([&] {
    auto* st = new Stepper();
    try {
      st->net = parse_network_spec(net_text);
      st->w = random_weights<float>(st->net, wseed);
      const Shape5 in{1, st->net.features_in, vec3::cube(e)};
      if (plan_mode == 0) {
        HostModel host;
        host.env.workers = double(g_workers);
        SearchBounds b;
        b.min_extent = e;
        b.max_extent = e;
        const PlanOutcome po = optimize_plan(st->net, host, b);
        require(po.feasible(), "ref_stepper: the reference planner found no plan");
        st->plan = *po.plan;
        require(st->plan.theta == i64(st->net.layers.size()), "ref_stepper: host-only plan expected");
      } else {
        st->plan = host_plan(st->net, in, conv_kind, 1);
      }
      st->input = Tensor5<float>(st->plan.input);
      std::mt19937_64 rng(iseed);
      std::uniform_real_distribution<double> d(-1.0, 1.0);
      for (i64 i = 0; i < st->input.size(); ++i) st->input.data()[i] = static_cast<float>(d(rng));
      i64 c = 0;
      for (size_t i = 0; i < st->net.layers.size(); ++i) {
        st->conv_at.push_back(std::holds_alternative<ConvSpec>(st->net.layers[i]) ? c++ : -1);
        if (const auto* p = std::get_if<PoolSpec>(&st->net.layers[i]))
          if (st->plan.layers[i].kind == PrimitiveKind::pool_fragments) st->windows.push_back(p->window);
        if (kinds) kinds[i] = static_cast<int>(st->plan.layers[i].kind);
      }
      st->cur = Tensor5<float>(st->input);
    } catch (...) {
      delete st;
      throw;
    }
    *handle = st;
  });
}

// Runs the next layer (the last one includes recombine_fragments).  *layer =
// the layer run, *seconds = its wall time, *done = 1 when it completed a
// forward (the next step starts a new forward from the same input).
int ref_stepper_step(void* handle, int64_t* layer, double* seconds, int* done) {
  return guard([&] {
    auto* st = static_cast<Stepper*>(handle);
    if (st->need_input) {  // outside the timed step, as measure_throughput copies its input
      st->cur = Tensor5<float>(st->input);
      st->need_input = false;
    }
    const auto t0 = std::chrono::steady_clock::now();
    const size_t li = st->li;
    const LayerPlan& lp = st->plan.layers[li];
    LayerContext<float> ctx = host_ctx();
    if (std::holds_alternative<ConvSpec>(st->net.layers[li])) {
      const ConvLayerParams<float>& p = st->w.convs[size_t(st->conv_at[li])];
      switch (lp.kind) {  // PlanRunner::host_conv (execute.hpp:281-297)
        case PrimitiveKind::direct_naive:
          st->cur = conv_direct(std::move(st->cur), p, ctx, DirectVariant::naive).output;
          break;
        case PrimitiveKind::direct_temp:
          st->cur = conv_direct(std::move(st->cur), p, ctx, DirectVariant::temp_buffer).output;
          break;
        case PrimitiveKind::fft_data_parallel:
          st->cur = conv_fft_data_parallel(std::move(st->cur), p, ctx).output;
          break;
        case PrimitiveKind::fft_task_parallel:
          st->cur = conv_fft_task_parallel(std::move(st->cur), p, ctx).output;
          break;
        case PrimitiveKind::fft_staged:
          st->cur = conv_fft_staged(std::move(st->cur), p, ctx).output;
          break;
        default: throw std::invalid_argument("ref_stepper: not a host convolution primitive");
      }
    } else {  // PlanRunner::pool (execute.hpp:312-317)
      const vec3 win = std::get<PoolSpec>(st->net.layers[li]).window;
      st->cur = lp.kind == PrimitiveKind::pool_fragments ? mpf_pool(std::move(st->cur), win, ctx).output
                                                         : max_pool(std::move(st->cur), win, ctx).output;
    }
    const bool last = li + 1 == st->net.layers.size();
    if (last && !st->windows.empty())  // PlanRunner::recombine (execute.hpp:219-226)
      st->cur = recombine_fragments(st->cur, st->windows, st->plan.input.s);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *layer = int64_t(li);
    *done = last ? 1 : 0;
    st->li = last ? 0 : li + 1;
    st->need_input = last;
  });
}

// the dense output of the last completed forward (valid until the next step)
int ref_stepper_output(void* handle, float* out, int64_t* shape5) {
  return guard([&] {
    auto* st = static_cast<Stepper*>(handle);
    const Shape5 s = st->cur.shape();
    if (shape5) {
      shape5[0] = s.s; shape5[1] = s.f; shape5[2] = s.n.x; shape5[3] = s.n.y; shape5[4] = s.n.z;
    }
    if (out) std::memcpy(out, st->cur.data(), sizeof(float) * size_t(st->cur.size()));
  });
}

int ref_stepper_free(void* handle) {
  delete static_cast<Stepper*>(handle);
  return 0;
}

}  // extern "C"
