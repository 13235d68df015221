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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <map>
#include <tuple>

#include "forward.hpp"

namespace vxg {

namespace {

// bytes of one batch entry at layer boundary li (z rows padded to the plan's pitch)
int64_t entry_bytes(const ForwardPlan& p, size_t li) {
  const Shape& s = p.shapes[li];
  return s.f * s.n.x * s.n.y * p.pz[li] * 4;
}

// VXG_SLAB_FUSION=0: fuse a first direct layer with its MPF by channel blocks
// instead of x slabs (A/B timing)
bool slab_fusion() {
  static const bool on = [] {
    const char* e = std::getenv("VXG_SLAB_FUSION");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return on;
}

}  // namespace

Model::Model(Ctx* ctx, const Net& n, const float* weights, bool device_ptr) : c(ctx), net(n) {
  net.validate();
  has_weights = weights != nullptr;
  int64_t f = net.fin, off = 0;
  int ci = 0;
  for (const auto& l : net.layers) {
    if (l.kind != 0) {
      conv_index.push_back(-1);
      continue;
    }
    conv_index.push_back(ci++);
    if (!has_weights) {
      f = l.fo;
      continue;
    }
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

ForwardPlan Model::plan(int64_t S, V3 e, const int* conv_algos, const int* pool_modes) const {
  ForwardPlan p;
  p.S = S;
  require(S > 0, "execute: batch must be positive");
  std::vector<int> modes;
  for (const auto& l : net.layers) {
    if (l.kind != 1) continue;
    int m = l.forced >= 0 ? l.forced : 1;
    if (pool_modes) {
      const int want = pool_modes[modes.size()];
      require(want == 0 || want == 1, "execute: pool mode must be plain (0) or fragments (1)");
      // planner.cpp:565-566
      require(l.forced < 0 || l.forced == want,
              "propagate_shapes: assignment conflicts with a forced pooling mode");
      m = want;
    }
    modes.push_back(m);
  }
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
      const Shape& pin = p.shapes[li];
      const double elems = double(pin.s * S) * double(pin.f) * double(pin.n.vol());
      p.choice[li].seconds = elems * (pool_elem > 0 ? pool_elem : 8.0 / 3e12);
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
    const V3 no{in.n.x - l.ext.x + 1, in.n.y - l.ext.y + 1, in.n.z - l.ext.z + 1};
    LayerChoice ch;
    bool fft_ok = true;
    double direct = 2.0 * double(B) * double(in.f) * double(l.fo) * double(no.vol()) *
                    double(l.ext.vol()) / 40e12;
    auto mit = measured.find(ci);
    try {
      ch.fft = plan_fft(in.n, l.ext, in.f, l.fo, B);
      if (mit != measured.end() && !mit->second.fft.empty()) {
        // measured-time choice of the tile size
        FftPlan best;
        double best_s = 1e300;
        for (const auto& kv : mit->second.fft) {
          FftPlan q = plan_fft(in.n, l.ext, in.f, l.fo, B, kv.first & kTuneT);
          if (kv.first & kTunePairTiles) q.quad = false;
          q.cost = kv.second.first + kv.second.second * double(B) * double(q.tiles);
          if (q.cost < best_s) {
            best_s = q.cost;
            best = q;
          }
        }
        ch.fft = best;
        ch.measured = true;
      }
    } catch (const invalid&) {
      fft_ok = false;
    }
    if (mit != measured.end() && mit->second.direct_vox > 0)
      direct = mit->second.direct_vox * double(B) * double(no.vol());
    if (algo == VXG_CONV_AUTO)
      algo = (fft_ok && ch.fft.cost < direct) ? VXG_CONV_FFT : VXG_CONV_DIRECT;
    ch.seconds = algo == VXG_CONV_FFT ? ch.fft.cost : direct;
    require(algo != VXG_CONV_FFT || fft_ok, "execute: kernel too large for the tiled FFT");
    ch.algo = algo;
    p.choice[li] = ch;
  }
  // Activations between layers get z rows padded to 16 bytes (every bundled
  // net's extents are odd all the way down), so row starts are aligned for
  // vector / bulk copies.  The input stays the caller's layout; plain max
  // pools (unpadded kernel) keep the whole forward unpadded.
  bool pitched = true;
  for (size_t li = 0; li < L; ++li)
    if (net.layers[li].kind == 1 && p.pool_mode[li] != 1) pitched = false;
  if (const char* e = std::getenv("VXG_NO_PITCH"))
    if (std::strcmp(e, "0") != 0) pitched = false;
  p.pz.resize(p.shapes.size());
  for (size_t i = 0; i < p.shapes.size(); ++i)
    p.pz[i] = (i == 0 || !pitched) ? p.shapes[i].n.z : (p.shapes[i].n.z + 3) / 4 * 4;
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

// Memory model of the executor.  A schedule is fixed by a target row count R
// for the FFT layers: a layer's useful group ("want") is the number of
// entries that gives its per-frequency contraction R rows (FFT conv) or that
// feeds the next layer's want (everything else), so upper levels never grab
// memory their own kernels do not profit from.  peak() is the exact high-water
// mark of running a subtree with that schedule, INCLUDING its input, which a
// level frees as soon as its last group has consumed it (ownership passes
// down the recursion).  At every level the executor takes the largest R whose
// subtree fits what the budget leaves (kTargets, R = 0: groups of one).
constexpr int64_t kTargets[] = {4096, 2048, 1024, 512, 256, 128, 64, 0};
constexpr int kNumTargets = sizeof(kTargets) / sizeof(kTargets[0]);

struct Sched {
  const Model& m;
  const ForwardPlan& p;
  size_t L;
  std::vector<std::vector<int64_t>> want;  // [target][layer]
  mutable std::map<std::tuple<int, size_t, int64_t, bool>, int64_t> memo;

  Sched(const Model& mm, const ForwardPlan& pp) : m(mm), p(pp), L(mm.net.layers.size()) {
    want.assign(kNumTargets, std::vector<int64_t>(L + 1, 1));
    for (int t = 0; t < kNumTargets; ++t)
      for (size_t li = L; li-- > 0;) {
        const Step st = step(li);
        const int64_t next = st.next < L ? want[size_t(t)][st.next] : 1;
        int64_t own = 1;
        const Layer& l = m.net.layers[li];
        if (l.kind == 0 && p.choice[li].algo == VXG_CONV_FFT && kTargets[t] > 0)
          own = (kTargets[t] + p.choice[li].fft.tiles - 1) / p.choice[li].fft.tiles;
        want[size_t(t)][li] = std::max(own, (next + st.P - 1) / st.P);
      }
  }

  Step step(size_t li) const {
    const Layer& l = m.net.layers[li];
    if (l.kind == 0 && p.choice[li].algo == VXG_CONV_DIRECT && li + 1 < L &&
        m.net.layers[li + 1].kind == 1 && p.pool_mode[li + 1] == 1)
      return Step{li, li + 2, true, m.net.layers[li + 1].ext.vol()};
    const int64_t P = (l.kind == 1 && p.pool_mode[li] == 1) ? l.ext.vol() : 1;
    return Step{li, li + 1, false, P};
  }

  int64_t in_bytes(size_t li, int64_t B) const { return li >= L ? 0 : B * entry_bytes(p, li); }

  int64_t out_bytes(const Step& st, int64_t g) const {
    if (st.next >= L) return 0;  // leaves write the final buffer
    return g * st.P * entry_bytes(p, st.next);
  }

  int64_t ws_bytes(const Step& st, int64_t g) const {
    const Layer& l = m.net.layers[st.li];
    if (st.fused) return g * std::min<int64_t>(16, l.fo) * entry_bytes(p, st.li + 1) / p.shapes[st.li + 1].f;
    if (l.kind != 0 || p.choice[st.li].algo != VXG_CONV_FFT) return 0;
    const LayerChoice& ch = p.choice[st.li];
    const int64_t M = g * ch.fft.tiles;
    return fft_chunk_bytes(ch.fft, p.shapes[st.li].f, l.fo, std::min<int64_t>(M, fft_reserved_rows()));
  }

  int64_t group_of(int t, size_t li, int64_t B) const { return std::min(B, want[size_t(t)][li]); }

  // high-water bytes of layers [li, L) on B entries (input included) under target t
  int64_t peak(int t, size_t li, int64_t B, bool freeable) const {
    if (li >= L || B <= 0) return 0;
    const auto key = std::make_tuple(t, li, B, freeable);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    const Step st = step(li);
    const int64_t G = group_of(t, li, B);
    const int64_t in = in_bytes(li, B);
    auto group = [&](int64_t g, bool last) {
      const int64_t run = in + out_bytes(st, g) + ws_bytes(st, g);
      const int64_t sub = peak(t, st.next, g * st.P, true);  // includes out(g)
      const int64_t keep = (last && freeable) ? 0 : in;
      return std::max(run, keep + sub);
    };
    int64_t r = group(G, G >= B);
    if (B % G) r = std::max(r, group(B % G, true));
    memo.emplace(key, r);
    return r;
  }

  // largest target whose subtree fits `avail` on top of the (already held) input
  int choose_target(size_t li, int64_t B, bool freeable, int64_t avail) const {
    for (int t = 0; t < kNumTargets; ++t)
      if (peak(t, li, B, freeable) - in_bytes(li, B) <= avail) return t;
    return kNumTargets - 1;
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

  int64_t avail() const { return m.c->avail(); }

  // run layers [li, L) on B entries of layer li's input at `in`; `owner`
  // (optional) holds the input and is released once the last group consumed it
  void run(size_t li, const float* in, int64_t B, DevBuf* owner) {
    const size_t L = m.net.layers.size();
    const Step st = sched.step(li);
    const int t = sched.choose_target(li, B, owner != nullptr, avail());
    const int64_t G = sched.group_of(t, li, B);
    if (trace_on())
      std::fprintf(stderr, "[vxg] layer %zu: %lld entries, target rows %lld, groups of %lld\n", li,
                   (long long)B, (long long)kTargets[t], (long long)G);
    const int64_t in_entry = entry_bytes(p, li) / 4;
    for (int64_t b0 = 0; b0 < B; b0 += G) {
      const int64_t g = std::min(G, B - b0);
      const bool leaf = st.next >= L;
      DevBuf out;
      float* dst;
      if (leaf) {
        dst = final_frags + final_off * (entry_bytes(p, p.shapes.size() - 1) / 4);
      } else {
        out.alloc(m.c, sched.out_bytes(st, g));
        dst = out.as<float>();
      }
      exec(st, in + b0 * in_entry, g, dst);
      if (owner && b0 + g >= B) owner->reset();  // stream-ordered free after the last reader
      if (leaf)
        final_off += g * st.P;
      else
        run(st.next, dst, g * st.P, &out);
    }
  }

  void exec(const Step& st, const float* in, int64_t g, float* dst) {
    const size_t li = st.li;
    const Layer& l = m.net.layers[li];
    const Shape& si = p.shapes[li];
    if (st.fused) {
      const Layer& pool = m.net.layers[li + 1];
      const Shape& mid = p.shapes[li + 1];
      const int ci = m.conv_index[li];
      // single input map and 2x2x2 windows: x slabs of the conv output with
      // every output map (so the tensor-core direct kernel sees all f' maps),
      // each slab pooled into its x range of the fragments.  A slab of xs
      // (odd) conv planes yields (xs - 1) / 2 pooled planes for all 8
      // offsets; consecutive slabs share one conv plane.
      const int64_t plane_bytes = mid.f * mid.n.y * p.pz[li + 1] * 4;  // one conv x plane, all maps
      int64_t xs = avail() / std::max<int64_t>(plane_bytes, 1);
      xs = std::min(xs, mid.n.x);
      if (xs % 2 == 0) xs -= 1;
      if (si.f == 1 && pool.ext.x == 2 && pool.ext.y == 2 && pool.ext.z == 2 && xs >= 3 && slab_fusion()) {
        DevBuf tmp(m.c, xs * plane_bytes);
        const int64_t mx_full = mid.n.x / 2;
        const V3 n_in = si.n;
        const int64_t in_entry = n_in.x * n_in.y * p.pz[li];                  // f = 1
        const int64_t out_entry = int64_t(pool.ext.vol()) * l.fo * mx_full * (mid.n.y / 2) * p.pz[li + 2];
        for (int64_t e = 0; e < g; ++e) {
          for (int64_t x0 = 0; x0 + 1 < mid.n.x; x0 += xs - 1) {
            const int64_t nxs = std::min(xs, mid.n.x - x0);  // odd: x0 even, mid.n.x odd
            int h = timer.begin(li);
            conv_direct_device(m.c, in + e * in_entry + x0 * n_in.y * p.pz[li], 1, 1,
                               V3{nxs + l.ext.x - 1, n_in.y, n_in.z}, m.kern[size_t(ci)].as<float>(), l.fo, l.ext,
                               m.bias[size_t(ci)].as<float>(), l.relu, tmp.as<float>(), p.pz[li], p.pz[li + 1]);
            timer.end(h);
            h = timer.begin(li + 1);
            launch_mpf(m.c, tmp.as<float>(), 1, l.fo, V3{nxs, mid.n.y, mid.n.z}, pool.ext, dst + e * out_entry, l.fo,
                       0, p.pz[li + 1], p.pz[li + 2], mx_full, x0 / 2);
            timer.end(h);
          }
        }
        return;
      }
      // otherwise direct conv one channel block at a time, each block pooled
      // straight into its channel slice of the MPF output
      const int64_t per_ch = g * mid.n.x * mid.n.y * p.pz[li + 1] * 4;
      int64_t cb = std::max<int64_t>(1, avail() / std::max<int64_t>(per_ch, 1));
      cb = std::min(cb, l.fo);
      if (cb >= 16) cb -= cb % 16;
      DevBuf tmp(m.c, cb * per_ch);
      const int64_t kvol = l.ext.vol();
      for (int64_t c0 = 0; c0 < l.fo; c0 += cb) {
        const int64_t n = std::min(cb, l.fo - c0);
        int h = timer.begin(li);
        conv_direct_device(m.c, in, g, si.f, si.n, m.kern[size_t(ci)].as<float>() + c0 * si.f * kvol,
                           n, l.ext, m.bias[size_t(ci)].as<float>() + c0, l.relu, tmp.as<float>(), p.pz[li],
                           p.pz[li + 1]);
        timer.end(h);
        h = timer.begin(li + 1);
        launch_mpf(m.c, tmp.as<float>(), g, n, mid.n, pool.ext, dst, l.fo, c0, p.pz[li + 1], p.pz[li + 2]);
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
                        m.bias[size_t(ci)].as<float>(), l.relu, dst, p.choice[li].fft, ws, 0, p.pz[li],
                        p.pz[li + 1]);
      } else {
        conv_direct_device(m.c, in, g, si.f, si.n, m.kern[size_t(ci)].as<float>(), l.fo, l.ext,
                           m.bias[size_t(ci)].as<float>(), l.relu, dst, p.pz[li], p.pz[li + 1]);
      }
    } else if (p.pool_mode[li] == 1) {
      launch_mpf(m.c, in, g, si.f, si.n, l.ext, dst, 0, 0, p.pz[li], p.pz[li + 1]);
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
  auto key = std::make_pair(ci, (T << 8) | (plan.tc ? 1 : 0) | (plan.tc && plan.quad ? 2 : 0) |
                                    (plan.tc && plan.quad && q_bf16_correction() ? 4 : 0));
  auto it = spectra.find(key);
  if (it != spectra.end()) return it->second.as<float2>();
  int64_t f = net.fin;
  for (size_t li = 0; li < net.layers.size(); ++li) {
    const Layer& l = net.layers[li];
    if (l.kind != 0) continue;
    if (conv_index[li] == ci) {
      DevBuf b(c, kernel_spectra_bytes(plan, f, l.fo));
      compute_kernel_spectra(c, T, plan.tc, plan.quad, kern[size_t(ci)].as<float>(), l.fo, f, l.ext,
                             b.as<float2>());
      auto res = spectra.emplace(key, std::move(b));
      return res.first->second.as<float2>();
    }
    f = l.fo;
  }
  throw invalid("model: unknown conv layer");
}

int64_t Model::plan_bytes(const ForwardPlan& p, bool cache, int64_t target_rows) const {
  Sched s(*this, p);
  int t = kNumTargets - 1;
  for (int i = 0; i < kNumTargets; ++i)
    if (kTargets[i] <= target_rows) {
      t = i;
      break;
    }
  const int64_t in = p.S * entry_bytes(p, 0);
  const int64_t frags = p.S * p.alpha * entry_bytes(p, p.shapes.size() - 1);
  const int64_t dense = p.S * p.f_out * p.dense.vol() * 4;
  int64_t spectra_bytes = 0, scratch = 0;
  (void)cache;  // spectra are resident for the whole forward either way
  {
    int64_t f = net.fin;
    for (size_t li = 0; li < net.layers.size(); ++li) {
      const Layer& l = net.layers[li];
      if (l.kind != 0) continue;
      if (p.choice[li].algo == VXG_CONV_FFT) {
        const FftPlan& fp = p.choice[li].fft;
        spectra_bytes += kernel_spectra_bytes(fp, f, l.fo);
        // raw spectra before the tensor-core split (transient, one layer at a time)
        if (fp.tc) scratch = std::max(scratch, tile_nwp(fp.T, 16) * l.fo * f * 8);
      }
      f = l.fo;
    }
  }
  return frags + dense + spectra_bytes + scratch + std::max(in, s.peak(t, 0, p.S, false));
}

void Model::forward(const ForwardPlan& p, const float* d_in, float* d_dense, bool cache,
                    std::vector<double>* layer_seconds, cudaEvent_t before_output) {
  require(has_weights, "execute: planning-only model has no weights");
  EventTimer timer(c->stream, layer_seconds != nullptr);
  auto all_spectra = [&] {
    for (size_t li = 0; li < net.layers.size(); ++li)
      if (net.layers[li].kind == 0 && p.choice[li].algo == VXG_CONV_FFT) {
        const int h = timer.begin(li);
        spectra_for(conv_index[li], p.choice[li].fft, cache);
        timer.end(h);
      }
  };
  // cached kernel spectra outlive the forward: they come from the pool, first
  if (cache) all_spectra();
  // Everything else -- the final fragment tensor, per-forward kernel spectra
  // and their scratch, the recursion's activations and spectrum chunks --
  // lives in one arena block.  The block is kept between forwards (Ctx::held):
  // a freed block of that size is split by the pool for smaller requests,
  // after which the next forward's block no longer fits and the pool trims
  // and remaps ~100 GB; with every per-forward allocation inside it, the
  // steady state never touches the pool.
  const int64_t frags_bytes = p.S * p.alpha * entry_bytes(p, p.shapes.size() - 1);
  int64_t spec_bytes = 0, spec_scratch = 0;
  if (!cache) {
    int64_t f = net.fin;
    for (size_t li = 0; li < net.layers.size(); ++li) {
      const Layer& l = net.layers[li];
      if (l.kind != 0) continue;
      if (p.choice[li].algo == VXG_CONV_FFT) {
        const FftPlan& fp = p.choice[li].fft;
        spec_bytes += kernel_spectra_bytes(fp, f, l.fo) + 4096;
        if (fp.tc) spec_scratch = std::max(spec_scratch, tile_nwp(fp.T, 16) * l.fo * f * 8 + 4096);
      }
      f = l.fo;
    }
  }
  {
    Sched sched(*this, p);
    // the held block (if any) is ours to reuse: device memory in use but not
    // charged while idle
    const int64_t held = c->held_bytes;
    const int64_t avail0 = std::min(c->avail(), c->device_free() + held - (int64_t(512) << 20));
    const int64_t in0 = sched.in_bytes(0, p.S);
    const int64_t top = sched.peak(0, 0, p.S, false) - in0;
    const int64_t fixed = frags_bytes + 4096 + spec_bytes + spec_scratch;
    int64_t arena_bytes = int64_t(double(avail0) * 0.995);
    if (fixed + top <= avail0)
      arena_bytes = std::min(arena_bytes, fixed + top + top / 4 + (int64_t(256) << 20));
    if (trace_on())
      std::fprintf(stderr, "[vxg] forward arena: need %lld held %lld avail %lld (budget left %lld, device %lld)\n",
                   (long long)arena_bytes, (long long)held, (long long)avail0, (long long)c->avail(),
                   (long long)c->device_free());
    bool reuse = false;
    {
      std::lock_guard<std::mutex> lk(c->mu);  // release_idle_memory may drop an idle block
      if (c->held && c->held_bytes >= arena_bytes && c->held_bytes <= avail0) {
        reuse = true;
        arena_bytes = c->held_bytes;
        c->held_busy = true;
      }
    }
    if (reuse) {
      try {
        c->charge(arena_bytes);
      } catch (...) {
        std::lock_guard<std::mutex> lk(c->mu);
        c->held_busy = false;
        throw;
      }
    } else {
      c->drop_held();
      DevBuf blk(c, arena_bytes);  // charged
      std::lock_guard<std::mutex> lk(c->mu);
      c->held = blk.release_ptr();
      c->held_bytes = arena_bytes;
      c->held_busy = true;
    }
    struct Busy {
      Ctx* c;
      ~Busy() {
        c->release(c->held_bytes);  // idle: kept, not charged
        std::lock_guard<std::mutex> lk(c->mu);
        c->held_busy = false;
      }
    } busy{c};
    Arena arena;
    arena.reset(c->held, arena_bytes);
    struct Scope {
      Ctx* c;
      ~Scope() {
        std::lock_guard<std::mutex> lk(c->mu);
        c->arena = nullptr;
      }
    } scope{c};
    {
      std::lock_guard<std::mutex> lk(c->mu);
      c->arena = &arena;
    }
    DevBuf frags(c, frags_bytes);
    if (!cache) all_spectra();  // in the arena, so the group sizes below see their footprint
    {
      Runner r{*this, p, cache, Sched(*this, p), frags.as<float>(), 0, timer};
      r.run(0, d_in, p.S, nullptr);
    }
    if (!cache) spectra.clear();  // back to the arena (stream-ordered reuse only)
    const size_t nwin = p.windows.size() / 3;
    const Shape& fin = p.shapes.back();
    if (before_output) VXG_CUDA_CHECK(cudaStreamWaitEvent(c->stream, before_output, 0));
    if (nwin == 0) {
      VXG_CUDA_CHECK(cudaMemcpy2DAsync(d_dense, size_t(fin.n.z) * 4, frags.get(), size_t(p.pz.back()) * 4,
                                       size_t(fin.n.z) * 4, size_t(p.S * fin.f * fin.n.x * fin.n.y),
                                       cudaMemcpyDeviceToDevice, c->stream));
    } else {
      launch_recombine(c, frags.as<float>(), p.S * p.alpha, 0, fin.f, fin.n, p.windows.data(),
                       int(nwin), d_dense, p.S, p.pz.back());
    }
    arena_slack = arena_bytes - arena.peak;
  }
  timer.collect(layer_seconds, net.layers.size());
}

namespace {

double time_on_stream(Ctx* c, const std::function<void()>& fn, int reps) {
  cudaEvent_t a, b;
  VXG_CUDA_CHECK(cudaEventCreate(&a));
  VXG_CUDA_CHECK(cudaEventCreate(&b));
  fn();  // warm (first launch configures the kernel)
  double best = 1e300;
  for (int r = 0; r < reps; ++r) {
    VXG_CUDA_CHECK(cudaEventRecord(a, c->stream));
    fn();
    VXG_CUDA_CHECK(cudaEventRecord(b, c->stream));
    VXG_CUDA_CHECK(cudaEventSynchronize(b));
    float ms = 0.f;
    VXG_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, double(ms) * 1e-3);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

__global__ void fill_sample_kernel(float* x, int64_t n, uint32_t seed) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u ^ seed;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    x[i] = float(h & 0xFFFFFF) * (2.0f / 16777216.0f) - 1.0f;
  }
}

void fill_sample(Ctx* c, float* x, int64_t n, uint32_t seed) {
  fill_sample_kernel<<<grid_for(n, 256, int64_t(c->num_sms) * 8), 256, 0, c->stream>>>(x, n, seed);
  check_launch("fill_sample_kernel");
}

}  // namespace

// Measured-time planning (the reference's modelled seconds,
// cost.cpp:52-78 / planner.cpp:70-86, replaced by timed kernels): for every
// conv layer of the plan of (S, e), each admissible tile size T is timed on a
// sample of the layer's own (f, fo, k) -- ~216 rows, 3 tiles per axis -- and
// recorded as seconds per row; the direct kernel is timed too where the
// model's estimate is within 4x of the FFT's.  plan() then scales the
// per-row costs by each candidate's row count for the real extent.
// Measured costs can be saved (VXG_TUNE_SAVE=<file>) and replayed
// (VXG_TUNE_FILE=<file>) so that a profiled run (under ncu every launch is
// serialised and timings are meaningless) executes the plan of a normal run.
// One line per conv layer: "conv f fo kx ky kz direct_vox pool_elem {T fixed per_row}".
namespace {
std::string tune_key(int64_t f, int64_t fo, V3 k) {
  return std::to_string(f) + " " + std::to_string(fo) + " " + std::to_string(k.x) + " " +
         std::to_string(k.y) + " " + std::to_string(k.z);
}
}  // namespace

void Model::tune(int64_t S, V3 e) {
  require(has_weights, "tune: planning-only model has no weights");
  const ForwardPlan p0 = plan(S, e, nullptr);
  std::map<std::string, LayerCosts> replay;
  double replay_pool = -1;
  if (const char* fn = std::getenv("VXG_TUNE_FILE")) {
    if (FILE* fp = std::fopen(fn, "r")) {
      char line[4096];
      while (std::fgets(line, sizeof(line), fp)) {
        long long f, fo, kx, ky, kz;
        double dv, pe;
        int off = 0;
        if (std::sscanf(line, "conv %lld %lld %lld %lld %lld %lf %lf%n", &f, &fo, &kx, &ky, &kz, &dv, &pe,
                        &off) != 7)
          continue;
        LayerCosts lc;
        lc.direct_vox = dv;
        replay_pool = pe;
        const char* q = line + off;
        int T, n = 0;
        double a0, a1;
        while (std::sscanf(q, "%d %lf %lf%n", &T, &a0, &a1, &n) == 3) {
          lc.fft[T] = {a0, a1};
          q += n;
        }
        replay[tune_key(f, fo, V3{kx, ky, kz})] = lc;
      }
      std::fclose(fp);
    }
  }
  for (size_t li = 0; li < net.layers.size(); ++li) {
    const Layer& l = net.layers[li];
    if (l.kind != 0) continue;
    const int ci = conv_index[li];
    if (measured.count(ci)) continue;
    const Shape& in = p0.shapes[li];
    const int64_t f = in.f, fo = l.fo;
    const V3 k = l.ext;
    auto rit = replay.find(tune_key(f, fo, k));
    if (rit != replay.end()) {
      measured[ci] = rit->second;
      if (replay_pool > 0) pool_elem = replay_pool;
      continue;
    }
    LayerCosts lc;
    const float* w = kern[size_t(ci)].as<float>();
    const float* b = bias[size_t(ci)].as<float>();
    for (int ti = 0; ti < kNumTileSizes; ++ti) {
      const int T = kTileSizes[ti];
      if (T < k.x || T < k.y || T < k.z || T < 8) continue;
      V3 ns{3 * (T - k.x + 1) + k.x - 1, 3 * (T - k.y + 1) + k.y - 1, 3 * (T - k.z + 1) + k.z - 1};
      const V3 nso{ns.x - k.x + 1, ns.y - k.y + 1, ns.z - k.z + 1};
      // two sample sizes (~8 and ~40 entries of 27 tiles, the larger capped at
      // ~12 GB of sample data) -> fixed seconds per launch + seconds per row
      const int64_t per_entry = (f * ns.vol() + fo * nso.vol()) * 4 +
                                27 * (f + fo) * tile_nwp(T, 16) * 8;
      const int64_t S2 = std::max<int64_t>(9, std::min<int64_t>(40, (int64_t(12) << 30) / per_entry));
      const int64_t S1 = std::max<int64_t>(1, S2 / 5);
      FftPlan fp = plan_fft(ns, k, f, fo, S2, T);
      DevBuf x(c, S2 * f * ns.vol() * 4);
      DevBuf y(c, S2 * fo * nso.vol() * 4);
      fill_sample(c, x.as<float>(), S2 * f * ns.vol(), 12345u + uint32_t(T));
      // tensor-core layers: both tile shapes (quad frequencies x half the
      // maps, pairs x all maps) -- which wins depends on T and the row count
      const int variants = (fp.tc && fp.quad) ? 2 : 1;
      for (int vq = 0; vq < variants; ++vq) {
        fp.quad = fp.tc && fp.quad && vq == 0;
        DevBuf ws(c, kernel_spectra_bytes(fp, f, fo));
        compute_kernel_spectra(c, T, fp.tc, fp.quad, w, fo, f, k, ws.as<float2>());
        double t[2];
        const int64_t Ss[2] = {S1, S2};
        for (int q = 0; q < 2; ++q)
          t[q] = time_on_stream(c, [&] {
            conv_fft_device(c, x.as<float>(), Ss[q], f, ns, w, fo, k, b, l.relu, y.as<float>(), fp,
                            ws.as<float2>(), 0);
          }, 2);
        const double rows1 = double(S1 * fp.tiles), rows2 = double(S2 * fp.tiles);
        const double per_row = std::max(0.0, (t[1] - t[0]) / (rows2 - rows1));
        lc.fft[T | (vq ? kTunePairTiles : 0)] = {std::max(0.0, t[0] - per_row * rows1), per_row};
      }
    }
    // direct convolution, where it might compete
    {
      const LayerChoice& ch = p0.choice[li];
      const V3 no{in.n.x - k.x + 1, in.n.y - k.y + 1, in.n.z - k.z + 1};
      const double dmodel = 2.0 * double(f) * fo * double(no.vol()) * double(k.vol()) / 40e12;
      double best_fft = 1e300;
      for (const auto& kv : lc.fft) {
        const FftPlan q = plan_fft(in.n, k, f, fo, 1, kv.first & kTuneT);
        best_fft = std::min(best_fft, kv.second.first + kv.second.second * double(q.tiles));
      }
      if (ch.algo == VXG_CONV_DIRECT || dmodel < 4.0 * best_fft) {
        // a sample big enough to fill every SM several times over
        const int64_t d = f <= 8 ? 128 : 64;
        const V3 ns{d + k.x - 1, d + k.y - 1, d + k.z - 1};
        DevBuf x(c, f * ns.vol() * 4), y(c, fo * d * d * d * 4);
        fill_sample(c, x.as<float>(), f * ns.vol(), 777u);
        // followed by an MPF, the forward fuses the two: by x slabs with every
        // map (single input map, 2x2x2 windows), else by channel blocks whose
        // width the free memory sets (16 at the big patches the planner is
        // for); time the width the forward will use, since the kernel choice
        // depends on it
        const bool fused = li + 1 < p0.shapes.size() - 1 && net.layers[li + 1].kind == 1 &&
                           p0.pool_mode[li + 1] == 1;
        const V3 pw = fused ? net.layers[li + 1].ext : V3{0, 0, 0};
        const bool slabs = fused && f == 1 && pw.x == 2 && pw.y == 2 && pw.z == 2 && slab_fusion();
        const int64_t cb = fused && !slabs ? std::min<int64_t>(16, fo) : fo;
        const double t = time_on_stream(c, [&] {
          for (int64_t c0 = 0; c0 < fo; c0 += cb)
            conv_direct_device(c, x.as<float>(), 1, f, ns, w + c0 * f * k.vol(), std::min(cb, fo - c0), k,
                               b + c0, l.relu, y.as<float>() + c0 * d * d * d);
        }, 2);
        lc.direct_vox = t / double(d * d * d);
      }
    }
    if (trace_on()) {
      std::fprintf(stderr, "[vxg] tune layer %zu (f=%lld fo=%lld k=%lld):", li, (long long)f,
                   (long long)fo, (long long)k.x);
      for (const auto& kv : lc.fft)
        std::fprintf(stderr, " T%d%s %.3gms+%.3gns/row", kv.first & kTuneT, (kv.first & kTunePairTiles) ? "p" : "",
                     kv.second.first * 1e3, kv.second.second * 1e9);
      if (lc.direct_vox > 0) std::fprintf(stderr, " direct %.3gns/vox", lc.direct_vox * 1e9);
      std::fprintf(stderr, "\n");
    }
    measured[ci] = lc;
  }
  if (pool_elem < 0) {
    // MPF (p = 2) on a sample: seconds per input element
    const int64_t f = 80, n = 127;
    const V3 nv{n, n, n}, pw{2, 2, 2};
    DevBuf x(c, f * nv.vol() * 4), y(c, 8 * f * 63 * 63 * 63 * 4);
    fill_sample(c, x.as<float>(), f * nv.vol(), 99u);
    const double t = time_on_stream(c, [&] { launch_mpf(c, x.as<float>(), 1, f, nv, pw, y.as<float>()); }, 2);
    pool_elem = t / double(f * nv.vol());
  }
  if (const char* fn = std::getenv("VXG_TUNE_SAVE")) {
    if (FILE* fp = std::fopen(fn, "w")) {
      int64_t f = net.fin;
      for (size_t li = 0; li < net.layers.size(); ++li) {
        const Layer& l = net.layers[li];
        if (l.kind != 0) continue;
        const LayerCosts& lc = measured[conv_index[li]];
        std::fprintf(fp, "conv %s %.6e %.6e", tune_key(f, l.fo, l.ext).c_str(), lc.direct_vox, pool_elem);
        for (const auto& kv : lc.fft) std::fprintf(fp, " %d %.6e %.6e", kv.first, kv.second.first, kv.second.second);
        std::fprintf(fp, "\n");
        f = l.fo;
      }
      std::fclose(fp);
    }
  }
}

}  // namespace vxg
