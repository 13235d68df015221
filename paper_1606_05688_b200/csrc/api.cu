// The extern "C" boundary (include/vxg.h).  Every entry point converts the
// internal exceptions into the status codes that mirror the reference's
// error conventions, and handles host <-> device staging when mem == HOST.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "forward.hpp"
#include "linefft.hpp"

using namespace vxg;

namespace vxg {
namespace {
std::mutex g_ctx_mu;
std::vector<Ctx*> g_ctxs;
}  // namespace

void register_ctx(Ctx* c) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  g_ctxs.push_back(c);
}

void unregister_ctx(Ctx* c) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  g_ctxs.erase(std::remove(g_ctxs.begin(), g_ctxs.end(), c), g_ctxs.end());
}

void release_idle_memory(int device) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  for (Ctx* o : g_ctxs) {
    if (o->device != device) continue;
    o->drop_held();
    cudaStreamSynchronize(o->stream);
    cudaMemPoolTrimTo(o->pool, 0);
  }
}
}  // namespace vxg


namespace {

thread_local std::string g_err;
// device that was current when an entry point switched to its context's
// device (-1: none); guard() switches back on the way out
thread_local int g_prev_device = -1;

void use_device(int device) {
  int cur = 0;
  VXG_CUDA_CHECK(cudaGetDevice(&cur));
  if (cur == device) return;
  if (g_prev_device < 0) g_prev_device = cur;
  VXG_CUDA_CHECK(cudaSetDevice(device));
}

struct RestoreDevice {
  ~RestoreDevice() {
    if (g_prev_device >= 0) {
      cudaSetDevice(g_prev_device);
      g_prev_device = -1;
    }
  }
};

template <class F>
int guard(F&& f) {
  RestoreDevice restore;
  try {
    f();
    return VXG_OK;
  } catch (const parse_failure& e) {
    g_err = e.what();
    return VXG_PARSE;
  } catch (const invalid& e) {
    g_err = e.what();
    return VXG_INVALID;
  } catch (const exhausted& e) {
    g_err = e.what();
    return VXG_EXHAUSTED;
  } catch (const cuda_failure& e) {
    g_err = e.what();
    return VXG_CUDA;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return VXG_INVALID;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VXG_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw invalid(std::string(what) + ": null pointer");
}

// every entry point reaches its context through here: launches, streams and
// allocations then target the context's device whatever the thread's current one
Ctx* ctx_of(vxg_ctx* c) {
  if (!c) throw invalid("null context");
  Ctx* x = reinterpret_cast<Ctx*>(c);
  use_device(x->device);
  return x;
}

// Input view: a device pointer, staged from host when needed.
struct In {
  DevBuf buf;
  const float* p = nullptr;
  In(Ctx* c, int mem, const float* src, int64_t count) {
    if (mem == VXG_MEM_DEVICE) {
      p = src;
      return;
    }
    require(mem == VXG_MEM_HOST, "mem must be VXG_MEM_HOST or VXG_MEM_DEVICE");
    buf.alloc(c, count * 4);
    if (count > 0)
      VXG_CUDA_CHECK(cudaMemcpyAsync(buf.get(), src, size_t(count) * 4, cudaMemcpyHostToDevice, c->stream));
    p = buf.as<float>();
  }
};

// Output view: device pointer written in place, or a staging buffer copied
// back (and synchronised) by finish().
struct Out {
  DevBuf buf;
  float* p = nullptr;
  float* host = nullptr;
  int64_t count = 0;
  Out(Ctx* c, int mem, float* dst, int64_t n) : count(n) {
    if (mem == VXG_MEM_DEVICE) {
      p = dst;
      return;
    }
    buf.alloc(c, n * 4);
    p = buf.as<float>();
    host = dst;
  }
  void finish(Ctx* c) {
    if (host && count > 0)
      VXG_CUDA_CHECK(cudaMemcpyAsync(host, p, size_t(count) * 4, cudaMemcpyDeviceToHost, c->stream));
    if (host) VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  }
};

V3 v3_checked(const int64_t* a, const char* what) {
  need(a, what);
  return V3::of(a);
}

// audit: peak bytes of this call over the context's level at entry, in scalars
struct AuditScope {
  Ctx* c;
  int64_t base;
  int64_t saved_peak;
  explicit AuditScope(Ctx* ctx) : c(ctx) {
    std::lock_guard<std::mutex> lk(c->mu);
    base = c->current;
    saved_peak = c->peak;
    c->peak = c->current;
  }
  double peak_scalars() {
    std::lock_guard<std::mutex> lk(c->mu);
    return double(c->peak - base) / 4.0;
  }
  ~AuditScope() {
    std::lock_guard<std::mutex> lk(c->mu);
    if (saved_peak > c->peak) c->peak = saved_peak;
  }
};

}  // namespace

extern "C" {

const char* vxg_last_error(void) { return g_err.c_str(); }
const char* vxg_version(void) { return "vxg 0.1 (sm_100a)"; }

int vxg_ctx_create(int device, int64_t budget, vxg_ctx** out) {
  return guard([&] {
    need(out, "vxg_ctx_create");
    int count = 0;
    VXG_CUDA_CHECK(cudaGetDeviceCount(&count));
    require(device >= 0 && device < count, "vxg_ctx_create: no such CUDA device");
    VXG_CUDA_CHECK(cudaSetDevice(device));
    cudaDeviceProp prop{};
    VXG_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw cuda_failure("vxg is built for sm_100a (B200); device " + std::string(prop.name) +
                         " is sm_" + std::to_string(prop.major) + std::to_string(prop.minor));
    auto* c = new Ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    try {
      VXG_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      cudaMemPoolProps pp{};
      pp.allocType = cudaMemAllocationTypePinned;
      pp.location.type = cudaMemLocationTypeDevice;
      pp.location.id = device;
      VXG_CUDA_CHECK(cudaMemPoolCreate(&c->pool, &pp));
      uint64_t thresh = UINT64_MAX;
      VXG_CUDA_CHECK(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thresh));
      // other contexts' idle caches must not shrink this one's default budget
      release_idle_memory(device);
      size_t free_b = 0, total_b = 0;
      VXG_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
      // default budget: the HBM free at creation minus a 2.5 GiB reserve (CUDA
      // context growth, library workspaces, other allocators in the process)
      c->budget = budget > 0 ? budget : std::max<int64_t>(int64_t(free_b) - (int64_t(5) << 29), int64_t(free_b) / 2);
      VXG_CUDA_CHECK(cudaMalloc(&c->d_flag, sizeof(int)));
      VXG_CUDA_CHECK(cudaMemset(c->d_flag, 0, sizeof(int)));
      init_twiddles();
      init_line_fft(c);
    } catch (...) {
      if (c->stream) cudaStreamDestroy(c->stream);
      if (c->pool) cudaMemPoolDestroy(c->pool);
      delete c;
      throw;
    }
    register_ctx(c);
    *out = reinterpret_cast<vxg_ctx*>(c);
  });
}

int vxg_ctx_destroy(vxg_ctx* ctx) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    unregister_ctx(c);
    c->held_busy = false;
    c->drop_held();
    cudaStreamSynchronize(c->stream);
    if (c->d_flag) cudaFree(c->d_flag);
    cudaMemPoolDestroy(c->pool);
    cudaStreamDestroy(c->stream);
    delete c;
  });
}

int vxg_ctx_trim(vxg_ctx* ctx) {
  return guard([&] { release_idle_memory(ctx_of(ctx)->device); });
}

int vxg_ctx_sync(vxg_ctx* ctx) {
  return guard([&] { VXG_CUDA_CHECK(cudaStreamSynchronize(ctx_of(ctx)->stream)); });
}

int vxg_ctx_stream(vxg_ctx* ctx, void** s) {
  return guard([&] {
    need(s, "vxg_ctx_stream");
    *s = ctx_of(ctx)->stream;
  });
}

int vxg_ctx_memory(vxg_ctx* ctx, int64_t* current, int64_t* peak, int64_t* budget) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    if (current) *current = c->current;
    if (peak) *peak = c->peak;
    if (budget) *budget = c->budget;
  });
}

int vxg_ctx_reset_peak(vxg_ctx* ctx) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    c->peak = c->current;
  });
}

int64_t vxg_ctx_launches(vxg_ctx* ctx) { return ctx ? reinterpret_cast<Ctx*>(ctx)->launches.load() : -1; }

int vxg_ctx_profile(vxg_ctx* ctx, int enable) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    if (enable) {
      for (auto& r : c->krec) {
        c->spare_events.push_back(r.a);
        c->spare_events.push_back(r.b);
      }
      c->krec.clear();
    }
    c->prof = enable != 0;
  });
}

int vxg_ctx_kernel_stats(vxg_ctx* ctx, int kind, int64_t* launches, double* seconds,
                         double* flops, double* bytes) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    int64_t n = 0;
    double s = 0, fl = 0, by = 0;
    for (const auto& r : c->krec) {
      if (r.kind != kind) continue;
      float ms = 0;
      VXG_CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
      ++n;
      s += ms * 1e-3;
      fl += r.flops;
      by += r.bytes;
    }
    if (launches) *launches = n;
    if (seconds) *seconds = s;
    if (flops) *flops = fl;
    if (bytes) *bytes = by;
  });
}

int vxg_bench_ffma(vxg_ctx* ctx, double* tflops) {
  return guard([&] {
    need(tflops, "vxg_bench_ffma");
    *tflops = bench_ffma(ctx_of(ctx));
  });
}

// ---- layer primitives ---------------------------------------------------------

int vxg_conv(vxg_ctx* ctx, int algo, int mem, const float* in, int64_t S, int64_t f,
             const int64_t n_[3], const float* kernels, int64_t fo, const int64_t k_[3],
             const float* bias, int relu, float* out, vxg_audit* audit) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    const V3 n = v3_checked(n_, "vxg_conv: n"), k = v3_checked(k_, "vxg_conv: k");
    need(in, "vxg_conv: in");
    need(kernels, "vxg_conv: kernels");
    need(bias, "vxg_conv: bias");
    need(out, "vxg_conv: out");
    // ConvLayerParams::validate (layers.hpp:28-33) + Shape5::validate
    require(S > 0 && f > 0 && n.positive(), "Shape5: all extents must be positive");
    require(fo > 0 && k.positive(), "Shape5: all extents must be positive");
    require(k.x <= n.x && k.y <= n.y && k.z <= n.z, "conv: kernel larger than image");
    const V3 no{n.x - k.x + 1, n.y - k.y + 1, n.z - k.z + 1};
    AuditScope au(c);
    In xin(c, mem, in, S * f * n.vol());
    In win(c, mem, kernels, fo * f * k.vol());
    In bin(c, mem, bias, fo);
    Out o(c, mem, out, S * fo * no.vol());
    FftPlan plan;
    bool use_fft = algo == VXG_CONV_FFT;
    if (algo == VXG_CONV_AUTO || algo == VXG_CONV_FFT) {
      bool ok = true;
      try {
        plan = plan_fft(n, k, f, fo, S);
      } catch (const invalid&) {
        ok = false;
        if (algo == VXG_CONV_FFT) throw;
      }
      if (algo == VXG_CONV_AUTO) {
        const double direct =
            2.0 * double(S) * f * fo * double(no.vol()) * double(k.vol()) / 40e12;
        use_fft = ok && plan.cost < direct;
      }
    } else {
      require(algo == VXG_CONV_DIRECT, "vxg_conv: unknown algorithm");
    }
    // MemoryAudit (memory.hpp:100-103; the band of layers_test.cpp:388-414):
    // the working set is the call's tensors -- input, kernels, bias, output,
    // held by the caller (device) or staged here (host) -- plus the workspace.
    // Model: tensors + kernel spectra + max(raw-spectrum scratch of the
    // tensor-core split, the X / Y spectrum chunks of the rows used).
    const double tensors = double(S * f * n.vol() + fo * f * k.vol() + fo + S * fo * no.vol());
    double model = tensors;
    if (use_fft) {
      const int64_t rows = conv_fft_device(c, xin.p, S, f, n, win.p, fo, k, bin.p, relu != 0, o.p, plan, nullptr, 0);
      const double kspec = double(kernel_spectra_bytes(plan, f, fo)) / 4.0;
      const double raw = plan.tc ? double(tile_nwp(plan.T, 16) * fo * f * 8) / 4.0 : 0.0;
      const double chunks = double(fft_chunk_bytes(plan, f, fo, rows)) / 4.0;
      model += kspec + std::max(raw, chunks);
    } else {
      conv_direct_device(c, xin.p, S, f, n, win.p, fo, k, bin.p, relu != 0, o.p);
    }
    o.finish(c);
    if (audit) {
      VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
      audit->peak = au.peak_scalars() + (mem == VXG_MEM_DEVICE ? tensors : 0.0);
      audit->model = model;
    }
  });
}

int vxg_conv_fft_tiled(vxg_ctx* ctx, int mem, const float* in, int64_t S, int64_t f,
                       const int64_t n_[3], const float* kernels, int64_t fo, const int64_t k_[3],
                       const float* bias, int relu, float* out, int tile, int flags,
                       int64_t spectra_budget) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    const V3 n = v3_checked(n_, "vxg_conv_fft_tiled: n"), k = v3_checked(k_, "vxg_conv_fft_tiled: k");
    need(in, "vxg_conv_fft_tiled: in");
    need(kernels, "vxg_conv_fft_tiled: kernels");
    need(bias, "vxg_conv_fft_tiled: bias");
    need(out, "vxg_conv_fft_tiled: out");
    require(S > 0 && f > 0 && n.positive(), "Shape5: all extents must be positive");
    require(fo > 0 && k.positive(), "Shape5: all extents must be positive");
    require(k.x <= n.x && k.y <= n.y && k.z <= n.z, "conv: kernel larger than image");
    require(tile >= k.x && tile >= k.y && tile >= k.z, "vxg_conv_fft_tiled: tile smaller than the kernel");
    const V3 no{n.x - k.x + 1, n.y - k.y + 1, n.z - k.z + 1};
    const FftPlan plan = plan_fft_forced(n, k, f, fo, S, tile, !(flags & VXG_FFT_FFMA),
                                         !(flags & VXG_FFT_SINGLE_CTA));
    In xin(c, mem, in, S * f * n.vol());
    In win(c, mem, kernels, fo * f * k.vol());
    In bin(c, mem, bias, fo);
    Out o(c, mem, out, S * fo * no.vol());
    conv_fft_device(c, xin.p, S, f, n, win.p, fo, k, bin.p, relu != 0, o.p, plan, nullptr,
                    spectra_budget);
    o.finish(c);
  });
}

static int pool_common(vxg_ctx* ctx, int fragments, int mem, const float* in, int64_t S,
                       int64_t f, const int64_t n_[3], const int64_t p_[3], float* out,
                       vxg_audit* audit) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    const V3 n = v3_checked(n_, "pool: n"), p = v3_checked(p_, "pool: p");
    need(in, "pool: in");
    need(out, "pool: out");
    require(S > 0 && f > 0 && n.positive(), "Shape5: all extents must be positive");
    if (fragments) {
      require(p.positive(), "mpf_pool: window extents must be positive");
      require((n.x + 1) % p.x == 0 && (n.y + 1) % p.y == 0 && (n.z + 1) % p.z == 0,
              "mpf_pool: extent+1 must be divisible by the window");
    } else {
      require(p.positive(), "max_pool: window extents must be positive");
      require(n.x % p.x == 0 && n.y % p.y == 0 && n.z % p.z == 0,
              "max_pool: extents must be divisible by the window");
    }
    const V3 no{n.x / p.x, n.y / p.y, n.z / p.z};
    require(no.positive(), "Shape5: all extents must be positive");
    const int64_t P = fragments ? p.vol() : 1;
    AuditScope au(c);
    In xin(c, mem, in, S * f * n.vol());
    Out o(c, mem, out, S * P * f * no.vol());
    read_and_clear_flag(c);
    launch_nan_check(c, xin.p, S * f * n.vol());
    if (read_and_clear_flag(c))
      throw invalid(std::string(fragments ? "mpf_pool" : "max_pool") + ": NaN input rejected");
    if (fragments)
      launch_mpf(c, xin.p, S, f, n, p, o.p);
    else
      launch_maxpool(c, xin.p, S, f, n, p, o.p);
    o.finish(c);
    if (audit) {
      VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
      audit->peak = au.peak_scalars();
      audit->model = double(S * f * n.vol() + S * P * f * no.vol());  // pools row (cost.hpp:347)
      if (mem == VXG_MEM_DEVICE) audit->peak += audit->model;  // the caller's input and output
    }
  });
}

int vxg_max_pool(vxg_ctx* ctx, int mem, const float* in, int64_t S, int64_t f, const int64_t n[3],
                 const int64_t p[3], float* out, vxg_audit* audit) {
  return pool_common(ctx, 0, mem, in, S, f, n, p, out, audit);
}

int vxg_mpf_pool(vxg_ctx* ctx, int mem, const float* in, int64_t S, int64_t f, const int64_t n[3],
                 const int64_t p[3], float* out, vxg_audit* audit) {
  return pool_common(ctx, 1, mem, in, S, f, n, p, out, audit);
}

int vxg_recombine(vxg_ctx* ctx, int mem, const float* frag, int64_t Sf, int64_t f,
                  const int64_t n_[3], const int64_t* windows, int64_t nwin, int64_t S0,
                  float* dense) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    const V3 n = v3_checked(n_, "recombine: n");
    need(frag, "recombine: frag");
    need(dense, "recombine: dense");
    require(nwin >= 0 && (nwin == 0 || windows), "recombine_fragments: bad window");
    int64_t alpha = 1;
    V3 stride{1, 1, 1};
    for (int64_t w = 0; w < nwin; ++w) {
      const V3 wv = V3::of(windows + 3 * w);
      require(wv.positive(), "recombine_fragments: bad window");
      alpha *= wv.vol();
      for (int a = 0; a < 3; ++a) stride[a] *= wv[a];
    }
    require(S0 > 0 && Sf == S0 * alpha, "recombine_fragments: fragment batch mismatch");
    require(f > 0 && n.positive(), "Shape5: all extents must be positive");
    const int64_t count = Sf * f * n.vol();
    In xin(c, mem, frag, count);
    Out o(c, mem, dense, count);
    if (nwin == 0) {
      VXG_CUDA_CHECK(cudaMemcpyAsync(o.p, xin.p, size_t(count) * 4, cudaMemcpyDeviceToDevice, c->stream));
    } else {
      std::vector<int64_t> w(windows, windows + 3 * nwin);
      launch_recombine(c, xin.p, Sf, 0, f, n, w.data(), int(nwin), o.p, S0);
    }
    o.finish(c);
  });
}

// ---- transforms -----------------------------------------------------------------

int64_t vxg_optimal_fft_size(int64_t n, int profile) {
  if (n <= 0) {
    g_err = "optimal_fft_size: n must be positive";
    return -1;
  }
  static const int primes[6] = {2, 3, 5, 7, 11, 13};
  const int np = profile == VXG_PROFILE_DEVICE ? 4 : 6;
  for (int64_t m = n;; ++m) {
    int64_t r = m;
    int big = 0;
    for (int i = 0; i < np; ++i)
      while (r % primes[i] == 0) {
        r /= primes[i];
        if (primes[i] >= 11) ++big;
      }
    if (r == 1 && (profile != VXG_PROFILE_HOST || big <= 1)) return m;
  }
}

int vxg_fft_pruned_forward(vxg_ctx* ctx, int mem, const float* img, const int64_t n_[3],
                           const int64_t pad_[3], float* spec) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    const V3 n = v3_checked(n_, "fft: n"), pad = v3_checked(pad_, "fft: pad");
    need(img, "fft: img");
    need(spec, "fft: spec");
    require(n.positive(), "pruned fft: extents must be positive");
    require(pad.x >= n.x && pad.y >= n.y && pad.z >= n.z,
            "pruned fft: padded extents must cover the image");
    const int64_t count = (pad.x / 2 + 1) * pad.y * pad.z * 2;
    In xin(c, mem, img, n.vol());
    Out o(c, mem, spec, count);
    pruned_forward_device(c, xin.p, n, pad, reinterpret_cast<float2*>(o.p));
    o.finish(c);
  });
}

int vxg_fft_pruned_inverse(vxg_ctx* ctx, int mem, const float* spec, const int64_t pad_[3],
                           const int64_t crop_[3], float* out) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    const V3 pad = v3_checked(pad_, "fft: pad"), crop = v3_checked(crop_, "fft: crop");
    need(spec, "fft: spec");
    need(out, "fft: out");
    require(crop.positive(), "pruned fft: extents must be positive");
    require(pad.x >= crop.x && pad.y >= crop.y && pad.z >= crop.z,
            "pruned fft: padded extents must cover the image");
    const int64_t count = (pad.x / 2 + 1) * pad.y * pad.z * 2;
    In xin(c, mem, spec, count);
    Out o(c, mem, out, crop.vol());
    pruned_inverse_device(c, reinterpret_cast<const float2*>(xin.p), pad, crop, o.p);
    o.finish(c);
  });
}

int vxg_fft_batched_forward(vxg_ctx* ctx, int mem, const float* imgs, int64_t b,
                            const int64_t n_[3], const int64_t pad_[3], float* spec) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    const V3 n = v3_checked(n_, "fft: n"), pad = v3_checked(pad_, "fft: pad");
    need(imgs, "fft: imgs");
    need(spec, "fft: spec");
    require(b > 0, "batched fft: batch must be positive");
    require(n.positive(), "Shape5: all extents must be positive");
    require(pad.x >= n.x && pad.y >= n.y && pad.z >= n.z,
            "batched fft: padded extents must cover the image");
    const int64_t count = b * (pad.z / 2 + 1) * pad.y * pad.x * 2;
    In xin(c, mem, imgs, b * n.vol());
    Out o(c, mem, spec, count);
    batched_forward_device(c, xin.p, b, n, pad, reinterpret_cast<float2*>(o.p));
    o.finish(c);
  });
}

int vxg_fft_batched_inverse(vxg_ctx* ctx, int mem, const float* spec, int64_t b,
                            const int64_t pad_[3], const int64_t crop_[3], float* out) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    const V3 pad = v3_checked(pad_, "fft: pad"), crop = v3_checked(crop_, "fft: crop");
    need(spec, "fft: spec");
    need(out, "fft: out");
    require(b > 0 && crop.positive(), "batched inverse: bad region");
    require(pad.x >= crop.x && pad.y >= crop.y && pad.z >= crop.z,
            "batched inverse: region outside padded extents");
    const int64_t count = b * (pad.z / 2 + 1) * pad.y * pad.x * 2;
    In xin(c, mem, spec, count);
    Out o(c, mem, out, b * crop.vol());
    batched_inverse_device(c, reinterpret_cast<const float2*>(xin.p), b, pad, crop, o.p);
    o.finish(c);
  });
}

// ---- network description ------------------------------------------------------------

int vxg_net_parse(const char* text, vxg_net** out) {
  return guard([&] {
    need(text, "vxg_net_parse");
    need(out, "vxg_net_parse");
    auto* n = new vxg_net();
    try {
      n->net = parse_net(text);
    } catch (...) {
      delete n;
      throw;
    }
    *out = n;
  });
}

int vxg_net_free(vxg_net* net) {
  delete net;
  return VXG_OK;
}

int vxg_net_format(const vxg_net* net, char* buf, int64_t cap, int64_t* needed) {
  return guard([&] {
    need(net, "vxg_net_format");
    const std::string s = format_net(net->net);
    if (needed) *needed = int64_t(s.size()) + 1;
    if (buf && cap > 0) {
      const size_t nb = std::min<size_t>(size_t(cap - 1), s.size());
      std::memcpy(buf, s.data(), nb);
      buf[nb] = '\0';
    }
  });
}

int vxg_net_info(const vxg_net* net, int64_t info[5]) {
  return guard([&] {
    need(net, "vxg_net_info");
    need(info, "vxg_net_info");
    info[0] = int64_t(net->net.layers.size());
    info[1] = net->net.conv_count();
    info[2] = net->net.pool_count();
    info[3] = net->net.fin;
    info[4] = net->net.features_out();
  });
}

int vxg_net_layer(const vxg_net* net, int64_t l, int64_t* kind, int64_t ext[3], int64_t* fo,
                  int64_t* relu, int64_t* forced) {
  return guard([&] {
    need(net, "vxg_net_layer");
    require(l >= 0 && l < int64_t(net->net.layers.size()), "vxg_net_layer: index out of range");
    const Layer& L = net->net.layers[size_t(l)];
    if (kind) *kind = L.kind;
    if (ext) {
      ext[0] = L.ext.x;
      ext[1] = L.ext.y;
      ext[2] = L.ext.z;
    }
    if (fo) *fo = L.kind == 0 ? L.fo : 0;
    if (relu) *relu = L.relu ? 1 : 0;
    if (forced) *forced = L.forced;
  });
}

int vxg_net_fov(const vxg_net* net, int64_t fov[3]) {
  return guard([&] {
    need(net, "vxg_net_fov");
    need(fov, "vxg_net_fov");
    const V3 v = field_of_view(net->net);
    fov[0] = v.x;
    fov[1] = v.y;
    fov[2] = v.z;
  });
}

int vxg_net_propagate(const vxg_net* net, int64_t S, const int64_t e[3], const int* modes,
                      int64_t* shapes, int64_t* violation) {
  return guard([&] {
    need(net, "vxg_net_propagate");
    need(e, "vxg_net_propagate: e");
    need(shapes, "vxg_net_propagate: shapes");
    std::vector<int> m;
    if (modes) m.assign(modes, modes + net->net.pool_count());
    int64_t viol = -1;
    const auto chain = propagate_shapes(net->net, Shape{S, net->net.fin, V3::of(e)}, m, &viol);
    for (size_t i = 0; i < chain.size(); ++i) {
      shapes[5 * i + 0] = chain[i].s;
      shapes[5 * i + 1] = chain[i].f;
      shapes[5 * i + 2] = chain[i].n.x;
      shapes[5 * i + 3] = chain[i].n.y;
      shapes[5 * i + 4] = chain[i].n.z;
    }
    if (violation) *violation = viol;
  });
}

int64_t vxg_net_weight_count(const vxg_net* net) { return net ? net->net.weight_count() : -1; }

int vxg_random_weights(const vxg_net* net, uint64_t seed, float* w) {
  return guard([&] {
    need(net, "vxg_random_weights");
    need(w, "vxg_random_weights: weights");
    random_weights(net->net, seed, w);
  });
}

int vxg_fill_random(float* out, int64_t count, uint64_t seed) {
  return guard([&] {
    need(out, "vxg_fill_random");
    fill_random(out, count, seed);
  });
}

// ---- network forward ------------------------------------------------------------------

int vxg_model_create(vxg_ctx* ctx, const vxg_net* net, const float* weights, int mem,
                     vxg_model** out) {
  return guard([&] {
    Ctx* c = ctx_of(ctx);
    need(net, "vxg_model_create: net");
    need(out, "vxg_model_create: out");  // weights == NULL: planning-only model
    auto* m = new vxg_model();
    try {
      m->m = std::make_unique<Model>(c, net->net, weights, mem == VXG_MEM_DEVICE);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

int vxg_model_free(vxg_model* model) {
  return guard([&] {
    if (model) {
      use_device(model->m->c->device);
      cudaStreamSynchronize(model->m->c->stream);
      delete model;
    }
  });
}

int vxg_model_forward(vxg_model* model, int mem, const float* input, int64_t S, const int64_t e_[3],
                      const int* conv_algos, int cache_spectra, float* dense_out,
                      vxg_report* report) {
  return vxg_model_forward_ex(model, mem, input, S, e_, conv_algos, nullptr, cache_spectra, dense_out,
                              report);
}

int vxg_model_forward_ex(vxg_model* model, int mem, const float* input, int64_t S, const int64_t e_[3],
                         const int* conv_algos, const int* pool_modes, int cache_spectra,
                         float* dense_out, vxg_report* report) {
  return guard([&] {
    need(model, "vxg_model_forward: model");
    use_device(model->m->c->device);
    need(input, "vxg_model_forward: input");
    need(dense_out, "vxg_model_forward: dense_out");
    Model& m = *model->m;
    Ctx* c = m.c;
    const V3 e = v3_checked(e_, "vxg_model_forward: e");
    const ForwardPlan p = m.plan(S, e, conv_algos, pool_modes);
    AuditScope au(c);
    cudaEvent_t t0, t1;
    VXG_CUDA_CHECK(cudaEventCreate(&t0));
    VXG_CUDA_CHECK(cudaEventCreate(&t1));
    VXG_CUDA_CHECK(cudaEventRecord(t0, c->stream));
    In xin(c, mem, input, S * m.net.fin * e.vol());
    Out o(c, mem, dense_out, S * p.f_out * p.dense.vol());
    std::vector<double> layer_s;
    clear_flag_async(c);
    m.forward(p, xin.p, o.p, cache_spectra != 0, report ? &layer_s : nullptr);
    o.finish(c);
    VXG_CUDA_CHECK(cudaEventRecord(t1, c->stream));
    VXG_CUDA_CHECK(cudaEventSynchronize(t1));
    // the pools of the forward scan their inputs (check_no_nan, layers.hpp:111-116)
    if (read_and_clear_flag(c)) throw invalid("mpf_pool: NaN input rejected");
    float ms = 0;
    VXG_CUDA_CHECK(cudaEventElapsedTime(&ms, t0, t1));
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    if (report) {
      std::memset(report, 0, sizeof(*report));
      report->voxels = double(S) * double(p.dense.vol());
      report->seconds = ms * 1e-3;
      report->voxels_per_second = report->seconds > 0 ? report->voxels / report->seconds : 0;
      // the arena block is sized with headroom: audit what the forward used of it
      report->device_peak = au.peak_scalars() - double(m.arena_slack) / 4.0;
      report->layers = std::min<int64_t>(64, int64_t(layer_s.size()));
      for (int64_t i = 0; i < report->layers; ++i) report->layer_seconds[i] = layer_s[size_t(i)];
    }
  });
}

int vxg_model_forward_many(vxg_model* model, int64_t count, const float* const* inputs, int64_t S,
                           const int64_t e_[3], const int* conv_algos, int cache_spectra,
                           float* const* outputs, double* seconds) {
  return guard([&] {
    need(model, "vxg_model_forward_many: model");
    use_device(model->m->c->device);
    require(count >= 0, "vxg_model_forward_many: count must be >= 0");
    need(inputs, "vxg_model_forward_many: inputs");
    need(outputs, "vxg_model_forward_many: outputs");
    Model& m = *model->m;
    Ctx* c = m.c;
    const V3 e = v3_checked(e_, "vxg_model_forward_many: e");
    const ForwardPlan p = m.plan(S, e, conv_algos);
    const int64_t nin = S * m.net.fin * e.vol(), nout = S * p.f_out * p.dense.vol();
    for (int64_t k = 0; k < count; ++k) {
      need(inputs[k], "vxg_model_forward_many: input");
      need(outputs[k], "vxg_model_forward_many: output");
    }
    AuditScope au(c);
    // two copy streams (PCIe is full duplex) and double-buffered device tensors:
    // patch k + 1 uploads and patch k - 1 downloads while patch k runs
    struct Streams {
      cudaStream_t in = nullptr, out = nullptr;
      cudaEvent_t ev[8] = {};
      ~Streams() {
        for (auto& x : ev)
          if (x) cudaEventDestroy(x);
        if (in) cudaStreamDestroy(in);
        if (out) cudaStreamDestroy(out);
      }
    } st;
    VXG_CUDA_CHECK(cudaStreamCreateWithFlags(&st.in, cudaStreamNonBlocking));
    VXG_CUDA_CHECK(cudaStreamCreateWithFlags(&st.out, cudaStreamNonBlocking));
    for (auto& x : st.ev) VXG_CUDA_CHECK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    cudaEvent_t* h2d_done = st.ev;      // [2]
    cudaEvent_t* fwd_done = st.ev + 2;  // [2]
    cudaEvent_t* d2h_done = st.ev + 4;  // [2]
    // double buffering only if the forward still fits next to the second pair
    // of patch buffers (plan_bytes counts one input and one output)
    const int64_t one = (nin + nout) * 4;
    const int64_t need = m.plan_bytes(p, cache_spectra != 0, 0);
    const int64_t room = std::min(c->avail(), c->device_free() - (int64_t(512) << 20));
    const int nbuf = (count > 1 && need + one <= room) ? 2 : 1;
    DevBuf din[2], dout[2];
    for (int b = 0; b < nbuf && b < count; ++b) {
      din[b].alloc(c, nin * 4);
      dout[b].alloc(c, nout * 4);
    }
    VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));  // buffers exist before the copy streams use them
    cudaEvent_t t0, t1;
    VXG_CUDA_CHECK(cudaEventCreate(&t0));
    VXG_CUDA_CHECK(cudaEventCreate(&t1));
    VXG_CUDA_CHECK(cudaEventRecord(t0, c->stream));
    VXG_CUDA_CHECK(cudaStreamWaitEvent(st.in, t0, 0));
    auto h2d = [&](int64_t k) {
      const int b = int(k % nbuf);
      if (k >= nbuf) VXG_CUDA_CHECK(cudaStreamWaitEvent(st.in, fwd_done[b], 0));
      VXG_CUDA_CHECK(cudaMemcpyAsync(din[b].get(), inputs[k], size_t(nin) * 4, cudaMemcpyHostToDevice, st.in));
      VXG_CUDA_CHECK(cudaEventRecord(h2d_done[b], st.in));
    };
    clear_flag_async(c);
    if (count > 0) h2d(0);
    for (int64_t k = 0; k < count; ++k) {
      const int b = int(k % nbuf);
      if (nbuf == 2 && k + 1 < count) h2d(k + 1);  // prefetch under this forward
      VXG_CUDA_CHECK(cudaStreamWaitEvent(c->stream, h2d_done[b], 0));
      // the download of the patch that used this output buffer only has to end
      // before this forward writes its dense output: it runs under the forward
      m.forward(p, din[b].as<float>(), dout[b].as<float>(), cache_spectra != 0, nullptr,
                k >= nbuf ? d2h_done[b] : nullptr);
      VXG_CUDA_CHECK(cudaEventRecord(fwd_done[b], c->stream));
      VXG_CUDA_CHECK(cudaStreamWaitEvent(st.out, fwd_done[b], 0));
      VXG_CUDA_CHECK(cudaMemcpyAsync(outputs[k], dout[b].get(), size_t(nout) * 4, cudaMemcpyDeviceToHost,
                                     st.out));
      VXG_CUDA_CHECK(cudaEventRecord(d2h_done[b], st.out));
      if (nbuf == 1 && k + 1 < count) h2d(k + 1);  // single buffer: after this forward read it
    }
    VXG_CUDA_CHECK(cudaEventRecord(t1, st.out));
    VXG_CUDA_CHECK(cudaEventSynchronize(t1));
    VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    VXG_CUDA_CHECK(cudaEventElapsedTime(&ms, t0, t1));
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    if (seconds) *seconds = ms * 1e-3;
    if (read_and_clear_flag(c)) throw invalid("mpf_pool: NaN input rejected");
  });
}

int vxg_model_tune(vxg_model* model, int64_t S, const int64_t e[3]) {
  return guard([&] {
    need(model, "vxg_model_tune: model");
    use_device(model->m->c->device);
    model->m->tune(S, v3_checked(e, "vxg_model_tune: e"));
  });
}

int vxg_model_plan_info(vxg_model* model, int64_t S, const int64_t e[3], const int* conv_algos,
                        int64_t* out) {
  return guard([&] {
    need(model, "vxg_model_plan_info: model");
    use_device(model->m->c->device);
    need(out, "vxg_model_plan_info: out");
    const ForwardPlan p = model->m->plan(S, v3_checked(e, "vxg_model_plan_info: e"), conv_algos);
    for (size_t li = 0; li < model->m->net.layers.size(); ++li) {
      const bool conv = model->m->net.layers[li].kind == 0;
      const LayerChoice& ch = p.choice[li];
      const bool fft = conv && ch.algo == VXG_CONV_FFT;
      int64_t* o = out + 7 * li;
      o[0] = conv ? 0 : 1;
      o[1] = conv ? ch.algo : -1;
      o[2] = fft ? ch.fft.T : 0;
      o[3] = fft ? ch.fft.tiles : 0;
      o[4] = fft && ch.fft.tc ? (ch.fft.quad ? 1 : 2) : 0;  // 1: quad tiles, 2: pair tiles
      o[5] = ch.measured ? 1 : 0;
      o[6] = int64_t(ch.seconds * 1e9);
    }
  });
}

int vxg_model_plan_ex(vxg_model* model, int64_t S, const int64_t e[3], const int* conv_algos,
                      const int* pool_modes, int64_t* out, int64_t* bytes) {
  return guard([&] {
    need(model, "vxg_model_plan_ex: model");
    use_device(model->m->c->device);
    const Model& m = *model->m;
    const ForwardPlan p = m.plan(S, v3_checked(e, "vxg_model_plan_ex: e"), conv_algos, pool_modes);
    if (out)
      for (size_t li = 0; li < m.net.layers.size(); ++li) {
        const bool conv = m.net.layers[li].kind == 0;
        const LayerChoice& ch = p.choice[li];
        const bool fft = conv && ch.algo == VXG_CONV_FFT;
        int64_t* o = out + 8 * li;
        o[0] = conv ? 0 : 1;
        o[1] = conv ? ch.algo : p.pool_mode[li];
        o[2] = fft ? ch.fft.T : 0;
        o[3] = fft ? ch.fft.tiles : 0;
        o[4] = fft && ch.fft.tc ? (ch.fft.quad ? 1 : 2) : 0;  // 1: quad tiles, 2: pair tiles
        o[5] = ch.measured ? 1 : 0;
        o[6] = int64_t(ch.seconds * 1e9);
        o[7] = 0;
      }
    if (bytes) *bytes = m.plan_bytes(p, true);
  });
}

int64_t vxg_model_plan_bytes(vxg_model* model, int64_t S, const int64_t e[3], const int* algos) {
  int64_t r = -1;
  const int st = guard([&] {
    need(model, "vxg_model_plan_bytes");
    use_device(model->m->c->device);
    const ForwardPlan p = model->m->plan(S, V3::of(e), algos);
    r = model->m->plan_bytes(p, true);
  });
  return st == VXG_OK ? r : -1;
}

int vxg_net_forward(vxg_ctx* ctx, const vxg_net* net, const float* weights, int mem,
                    const float* input, int64_t S, const int64_t e[3], const int* conv_algos,
                    float* dense_out, vxg_report* report) {
  vxg_model* m = nullptr;
  int st = vxg_model_create(ctx, net, weights, mem, &m);
  if (st != VXG_OK) return st;
  st = vxg_model_forward(m, mem, input, S, e, conv_algos, 0, dense_out, report);
  const std::string keep = g_err;
  vxg_model_free(m);
  g_err = keep;
  return st;
}

}  // extern "C"
