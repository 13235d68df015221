// Device-resident network forward.
//
// Semantics follow execute_plan on an all-fragment plan
// (proj/include/voxin/execute.hpp:123-226, 388-402): layers run in order,
// every MPF multiplies the batch by the window volume, and the final
// fragments are recombined into the dense sliding-window output.  The
// execution order is depth-first over fragment groups: after an MPF layer the
// produced fragments are independent (batch separability, the idea behind
// run_suffix, execute.hpp:184-216), so the executor runs the rest of the
// network on the largest group of fragments that fits the HBM budget, frees
// it, and moves to the next group.  Groups are contiguous in the canonical
// batch order (s * P + offset at every pool), so the leaves write the final
// fragment tensor in exactly the order recombine_fragments expects.
#include <algorithm>
#include <cstring>

#include "forward.hpp"

namespace vxg {

namespace {

int64_t entry_bytes(const Shape& s) { return s.f * s.n.vol() * 4; }

}  // namespace

Model::Model(Ctx* ctx, const Net& n, const float* weights, bool device_ptr) : c(ctx), net(n) {
  net.validate();
  int64_t f = net.fin, off = 0;
  int ci = 0;
  for (const auto& l : net.layers) {
    if (l.kind != 0) {
      conv_index.push_back(-1);
      continue;
    }
    conv_index.push_back(ci++);
    const int64_t nk = l.fo * f * l.ext.vol();
    DevBuf kb(c, nk * 4), bb(c, l.fo * 4);
    const auto kind = device_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    VXG_CUDA_CHECK(cudaMemcpyAsync(kb.get(), weights + off, nk * 4, kind, c->stream));
    VXG_CUDA_CHECK(cudaMemcpyAsync(bb.get(), weights + off + nk, l.fo * 4, kind, c->stream));
    off += nk + l.fo;
    kern.push_back(std::move(kb));
    bias.push_back(std::move(bb));
    f = l.fo;
  }
  VXG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
}

ForwardPlan Model::plan(int64_t S, V3 e, const int* conv_algos) const {
  ForwardPlan p;
  p.S = S;
  require(S > 0, "execute: batch must be positive");
  std::vector<int> modes;
  for (const auto& l : net.layers)
    if (l.kind == 1) modes.push_back(l.forced >= 0 ? l.forced : 1);
  int64_t viol = -1;
  p.shapes = propagate_shapes(net, Shape{1, net.fin, e}, modes, &viol);
  require(viol < 0, "execute: plan input does not propagate through the network");
  const size_t L = net.layers.size();
  p.choice.resize(L);
  p.pool_mode.assign(L, -1);
  size_t pi = 0;
  for (size_t li = 0; li < L; ++li) {
    const Layer& l = net.layers[li];
    if (l.kind == 1) {
      p.pool_mode[li] = modes[pi++];
      if (p.pool_mode[li] == 1)
        for (int a = 0; a < 3; ++a) p.windows.push_back(l.ext[a]);
      continue;
    }
    const Shape& in = p.shapes[li];
    const int ci = conv_index[li];
    int algo = conv_algos ? conv_algos[ci] : VXG_CONV_AUTO;
    require(algo == VXG_CONV_AUTO || algo == VXG_CONV_DIRECT || algo == VXG_CONV_FFT,
            "execute: unknown convolution algorithm");
    const int64_t B = in.s * S;
    LayerChoice ch;
    bool fft_ok = true;
    try {
      ch.fft = plan_fft(in.n, l.ext, in.f, l.fo, B);
    } catch (const invalid&) {
      fft_ok = false;
    }
    if (algo == VXG_CONV_AUTO) {
      const V3 no{in.n.x - l.ext.x + 1, in.n.y - l.ext.y + 1, in.n.z - l.ext.z + 1};
      const double direct = 2.0 * double(B) * double(in.f) * double(l.fo) * double(no.vol()) *
                            double(l.ext.vol()) / 40e12;
      algo = (fft_ok && ch.fft.cost < direct) ? VXG_CONV_FFT : VXG_CONV_DIRECT;
    }
    require(algo != VXG_CONV_FFT || fft_ok, "execute: kernel too large for the tiled FFT");
    ch.algo = algo;
    p.choice[li] = ch;
  }
  const Shape& fin = p.shapes.back();
  p.f_out = fin.f;
  p.alpha = fin.s;
  V3 stride{1, 1, 1};
  for (size_t w = 0; w < p.windows.size() / 3; ++w)
    for (int a = 0; a < 3; ++a) stride[a] *= p.windows[3 * w + a];
  p.dense = V3{stride.x * fin.n.x, stride.y * fin.n.y, stride.z * fin.n.z};
  return p;
}

namespace {

// One execution step starting at layer li: a single layer, or a direct conv
// fused with the MPF that follows it (conv output produced and pooled one
// channel block at a time, so the full-resolution conv output never exists).
struct Step {
  size_t li, next;
  bool fused;
  int64_t P;  // entries produced per input entry
};

// Memory model of the executor.  need_min[li] is the peak (bytes, input of
// layer li excluded) of running layers [li, L) on ONE entry with groups of one
// entry everywhere below -- independent of the batch, so the greedy group
// choice at each level is a single binary search.
struct Sched {
  const Model& m;
  const ForwardPlan& p;
  bool cache;
  std::vector<int64_t> need_min;

  Sched(const Model& mm, const ForwardPlan& pp, bool c) : m(mm), p(pp), cache(c) {
    const size_t L = m.net.layers.size();
    need_min.assign(L + 1, 0);
    for (size_t li = L; li-- > 0;) {
      const Step st = step(li);
      // the P entries this makes are processed one at a time below
      need_min[li] = out_bytes(st, 1) + std::max(ws_bytes(st, 1), st.next < L ? need_min[st.next] : 0);
    }
  }

  Step step(size_t li) const {
    const size_t L = m.net.layers.size();
    const Layer& l = m.net.layers[li];
    if (l.kind == 0 && p.choice[li].algo == VXG_CONV_DIRECT && li + 1 < L &&
        m.net.layers[li + 1].kind == 1 && p.pool_mode[li + 1] == 1)
      return Step{li, li + 2, true, m.net.layers[li + 1].ext.vol()};
    const int64_t P = (l.kind == 1 && p.pool_mode[li] == 1) ? l.ext.vol() : 1;
    return Step{li, li + 1, false, P};
  }

  int64_t out_bytes(const Step& st, int64_t g) const {
    if (st.next >= m.net.layers.size()) return 0;  // leaves write the final buffer
    return g * st.P * entry_bytes(p.shapes[st.next]);
  }

  // channel block of the fused direct conv: multiple of 16 maps
  int64_t fused_block_bytes(const Step& st, int64_t g, int64_t cb) const {
    const Shape& mid = p.shapes[st.li + 1];
    return g * cb * mid.n.vol() * 4;
  }

  int64_t ws_bytes(const Step& st, int64_t g) const {
    const Layer& l = m.net.layers[st.li];
    if (st.fused) return fused_block_bytes(st, g, std::min<int64_t>(16, l.fo));
    if (l.kind != 0 || p.choice[st.li].algo != VXG_CONV_FFT) return 0;
    const LayerChoice& ch = p.choice[st.li];
    const Shape& in = p.shapes[st.li];
    const int64_t M = g * ch.fft.tiles;
    return fft_chunk_bytes(ch.fft, in.f, l.fo, std::min<int64_t>(M, 256));
  }

  int64_t group_need(const Step& st, int64_t g) const {
    const size_t L = m.net.layers.size();
    const int64_t rec = st.next < L ? need_min[st.next] : 0;
    return out_bytes(st, g) + std::max(ws_bytes(st, g), rec);
  }

  // largest group (entries of layer li's input) whose step fits `avail`
  int64_t choose(const Step& st, int64_t B, int64_t avail) const {
    if (group_need(st, B) <= avail) return B;
    int64_t lo = 1, hi = B;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (group_need(st, mid) <= avail)
        lo = mid;
      else
        hi = mid - 1;
    }
    return lo;
  }
};

struct EventTimer {
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  cudaStream_t s;
  bool on;
  EventTimer(cudaStream_t st, bool enabled) : s(st), on(enabled) {}
  int begin(size_t li) {
    if (!on) return -1;
    cudaEvent_t a, b;
    VXG_CUDA_CHECK(cudaEventCreate(&a));
    VXG_CUDA_CHECK(cudaEventCreate(&b));
    VXG_CUDA_CHECK(cudaEventRecord(a, s));
    ev.push_back({int(li), {a, b}});
    return int(ev.size()) - 1;
  }
  void end(int h) {
    if (h >= 0) VXG_CUDA_CHECK(cudaEventRecord(ev[size_t(h)].second.second, s));
  }
  void collect(std::vector<double>* out, size_t L) {
    if (!on) return;
    out->assign(L, 0.0);
    for (auto& e : ev) {
      float ms = 0.f;
      VXG_CUDA_CHECK(cudaEventSynchronize(e.second.second));
      VXG_CUDA_CHECK(cudaEventElapsedTime(&ms, e.second.first, e.second.second));
      (*out)[size_t(e.first)] += ms * 1e-3;
    }
  }
  ~EventTimer() {
    for (auto& e : ev) {
      cudaEventDestroy(e.second.first);
      cudaEventDestroy(e.second.second);
    }
  }
};

struct Runner {
  Model& m;
  const ForwardPlan& p;
  bool cache;
  Sched sched;
  float* final_frags;
  int64_t final_off = 0;
  EventTimer& timer;

  int64_t avail() const {
    std::lock_guard<std::mutex> lk(m.c->mu);
    return m.c->budget - m.c->current;
  }

  // run layers [li, L) on B entries of layer li's input at `in` (not owned)
  void run(size_t li, const float* in, int64_t B) {
    const size_t L = m.net.layers.size();
    const Step st = sched.step(li);
    const int64_t G = sched.choose(st, B, avail());
    const int64_t in_entry = entry_bytes(p.shapes[li]) / 4;
    for (int64_t b0 = 0; b0 < B; b0 += G) {
      const int64_t g = std::min(G, B - b0);
      const bool leaf = st.next >= L;
      DevBuf out;
      float* dst;
      if (leaf) {
        dst = final_frags + final_off * (entry_bytes(p.shapes.back()) / 4);
      } else {
        out.alloc(m.c, sched.out_bytes(st, g));
        dst = out.as<float>();
      }
      exec(st, in + b0 * in_entry, g, dst);
      if (leaf)
        final_off += g * st.P;
      else
        run(st.next, dst, g * st.P);
    }
  }

  void exec(const Step& st, const float* in, int64_t g, float* dst) {
    const size_t li = st.li;
    const Layer& l = m.net.layers[li];
    const Shape& si = p.shapes[li];
    if (st.fused) {
      // direct conv one channel block at a time, each block pooled straight
      // into its channel slice of the MPF output
      const Layer& pool = m.net.layers[li + 1];
      const Shape& mid = p.shapes[li + 1];
      const int ci = m.conv_index[li];
      const int64_t per_ch = g * mid.n.vol() * 4;
      int64_t cb = std::max<int64_t>(1, avail() / std::max<int64_t>(per_ch, 1));
      cb = std::min(cb, l.fo);
      if (cb >= 16) cb -= cb % 16;
      DevBuf tmp(m.c, cb * per_ch);
      const int64_t kvol = l.ext.vol();
      for (int64_t c0 = 0; c0 < l.fo; c0 += cb) {
        const int64_t n = std::min(cb, l.fo - c0);
        int h = timer.begin(li);
        conv_direct_device(m.c, in, g, si.f, si.n, m.kern[size_t(ci)].as<float>() + c0 * si.f * kvol,
                           n, l.ext, m.bias[size_t(ci)].as<float>() + c0, l.relu, tmp.as<float>());
        timer.end(h);
        h = timer.begin(li + 1);
        launch_mpf(m.c, tmp.as<float>(), g, n, mid.n, pool.ext, dst, l.fo, c0);
        timer.end(h);
      }
      return;
    }
    const int h = timer.begin(li);
    if (l.kind == 0) {
      const int ci = m.conv_index[li];
      if (p.choice[li].algo == VXG_CONV_FFT) {
        const float2* ws = m.spectra_for(ci, p.choice[li].fft, cache);
        conv_fft_device(m.c, in, g, si.f, si.n, m.kern[size_t(ci)].as<float>(), l.fo, l.ext,
                        m.bias[size_t(ci)].as<float>(), l.relu, dst, p.choice[li].fft, ws, 0);
      } else {
        conv_direct_device(m.c, in, g, si.f, si.n, m.kern[size_t(ci)].as<float>(), l.fo, l.ext,
                           m.bias[size_t(ci)].as<float>(), l.relu, dst);
      }
    } else if (p.pool_mode[li] == 1) {
      launch_mpf(m.c, in, g, si.f, si.n, l.ext, dst);
    } else {
      launch_maxpool(m.c, in, g, si.f, si.n, l.ext, dst);
    }
    timer.end(h);
  }
};

}  // namespace

// Kernel spectra are computed at a layer's first use in a forward and kept
// for the rest of it (every fragment group reuses them); without `cache`
// they are dropped at the end of the forward, so every forward recomputes them.
const float2* Model::spectra_for(int ci, const FftPlan& plan, bool /*cache*/) {
  const int T = plan.T;
  auto key = std::make_pair(ci, (T << 8) | (plan.tc ? 1 : 0));
  auto it = spectra.find(key);
  if (it != spectra.end()) return it->second.as<float2>();
  int64_t f = net.fin;
  for (size_t li = 0; li < net.layers.size(); ++li) {
    const Layer& l = net.layers[li];
    if (l.kind != 0) continue;
    if (conv_index[li] == ci) {
      DevBuf b(c, kernel_spectra_bytes(plan, f, l.fo));
      compute_kernel_spectra(c, T, plan.tc, kern[size_t(ci)].as<float>(), l.fo, f, l.ext,
                             b.as<float2>());
      auto res = spectra.emplace(key, std::move(b));
      return res.first->second.as<float2>();
    }
    f = l.fo;
  }
  throw invalid("model: unknown conv layer");
}

int64_t Model::plan_bytes(const ForwardPlan& p, bool cache) const {
  Sched s(*this, p, cache);
  const int64_t in = p.S * entry_bytes(p.shapes[0]);
  const int64_t frags = p.S * p.alpha * entry_bytes(p.shapes.back());
  const int64_t dense = p.S * p.f_out * p.dense.vol() * 4;
  int64_t spectra_bytes = 0;
  (void)cache;  // spectra are resident for the whole forward either way
  {
    int64_t f = net.fin;
    for (size_t li = 0; li < net.layers.size(); ++li) {
      const Layer& l = net.layers[li];
      if (l.kind != 0) continue;
      if (p.choice[li].algo == VXG_CONV_FFT) spectra_bytes += kernel_spectra_bytes(p.choice[li].fft, f, l.fo);
      f = l.fo;
    }
  }
  return in + frags + dense + spectra_bytes + s.need_min[0];
}

void Model::forward(const ForwardPlan& p, const float* d_in, float* d_dense, bool cache,
                    std::vector<double>* layer_seconds) {
  EventTimer timer(c->stream, layer_seconds != nullptr);
  DevBuf frags(c, p.S * p.alpha * entry_bytes(p.shapes.back()));
  // kernel spectra first, so the group sizes below see their footprint
  for (size_t li = 0; li < net.layers.size(); ++li)
    if (net.layers[li].kind == 0 && p.choice[li].algo == VXG_CONV_FFT) {
      const int h = timer.begin(li);
      spectra_for(conv_index[li], p.choice[li].fft, cache);
      timer.end(h);
    }
  Runner r{*this, p, cache, Sched(*this, p, cache), frags.as<float>(), 0, timer};
  r.run(0, d_in, p.S);
  if (!cache) spectra.clear();  // stream-ordered frees: recomputed by the next forward
  const size_t nwin = p.windows.size() / 3;
  if (nwin == 0) {
    VXG_CUDA_CHECK(cudaMemcpyAsync(d_dense, frags.get(), size_t(frags.bytes()),
                                   cudaMemcpyDeviceToDevice, c->stream));
  } else {
    const Shape& fin = p.shapes.back();
    launch_recombine(c, frags.as<float>(), p.S * p.alpha, 0, fin.f, fin.n, p.windows.data(),
                     int(nwin), d_dense, p.S);
  }
  timer.collect(layer_seconds, net.layers.size());
}

}  // namespace vxg
