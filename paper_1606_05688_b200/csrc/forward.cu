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

// Peak-memory model of running layers [li, L) on B entries (input included),
// with the executor's greedy group choice below each MPF.
struct PeakModel {
  const Model& m;
  const ForwardPlan& p;
  bool cache;

  int64_t conv_ws(size_t li, int64_t B) const {
    const LayerChoice& ch = p.choice[li];
    if (ch.algo != VXG_CONV_FFT) return 0;
    const Shape& in = p.shapes[li];
    const int64_t fo = m.net.layers[li].fo;
    const int64_t M = B * ch.fft.tiles;
    const int64_t rows = std::min<int64_t>(M, 256);
    int64_t ws = fft_chunk_bytes(ch.fft, in.f, fo, rows);
    if (!cache) ws += ch.fft.nwb * fo * in.f * 16 * 8;
    return ws;
  }

  int64_t peak(size_t li, int64_t B, int64_t avail) const {
    const size_t L = m.net.layers.size();
    if (li >= L) return 0;
    const int64_t in = B * entry_bytes(p.shapes[li]);
    const Layer& l = m.net.layers[li];
    const bool last = li + 1 == L;
    if (l.kind == 0) {
      const int64_t out = last ? 0 : B * entry_bytes(p.shapes[li + 1]);
      const int64_t here = in + out + conv_ws(li, B);
      const int64_t next = last ? 0 : peak(li + 1, B, avail);
      return std::max(here, next);
    }
    if (last) return in;
    if (p.pool_mode[li] == 0) {
      const int64_t out = B * entry_bytes(p.shapes[li + 1]);
      return std::max(in + out, peak(li + 1, B, avail));
    }
    const int64_t G = choose(li, B, avail);
    return in + peak(li + 1, G, avail - in);
  }

  // largest fragment group (output entries per pass) that fits `avail`
  int64_t choose(size_t li, int64_t B, int64_t avail) const {
    const int64_t total = B * m.net.layers[li].ext.vol();
    const int64_t in = B * entry_bytes(p.shapes[li]);
    const int64_t room = avail - in;
    if (peak(li + 1, total, room) <= room) return total;
    int64_t lo = 1, hi = total;
    if (peak(li + 1, 1, room) > room) return 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (peak(li + 1, mid, room) <= room)
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
  float* final_frags;
  int64_t final_off = 0;
  EventTimer& timer;

  float* final_slot() const {
    return final_frags + final_off * entry_bytes(p.shapes.back()) / 4;
  }

  void run(size_t li, const float* in, DevBuf* owner, int64_t B) {
    const size_t L = m.net.layers.size();
    const Layer& l = m.net.layers[li];
    const Shape& si = p.shapes[li];
    const Shape& so = p.shapes[li + 1];
    const bool last = li + 1 == L;
    if (l.kind == 0) {
      DevBuf out;
      float* dst = last ? final_slot() : nullptr;
      if (!last) {
        out.alloc(m.c, B * entry_bytes(so));
        dst = out.as<float>();
      }
      const int ci = m.conv_index[li];
      const int h = timer.begin(li);
      if (p.choice[li].algo == VXG_CONV_FFT) {
        const float2* ws = m.spectra_for(ci, p.choice[li].fft.T, cache);
        conv_fft_device(m.c, in, B, si.f, si.n, m.kern[size_t(ci)].as<float>(), l.fo, l.ext,
                        m.bias[size_t(ci)].as<float>(), l.relu, dst, p.choice[li].fft, ws, 0);
      } else {
        conv_direct_device(m.c, in, B, si.f, si.n, m.kern[size_t(ci)].as<float>(), l.fo, l.ext,
                           m.bias[size_t(ci)].as<float>(), l.relu, dst);
      }
      timer.end(h);
      if (owner) owner->reset();
      if (last) {
        final_off += B;
        return;
      }
      run(li + 1, dst, &out, B);
      return;
    }
    // pooling
    if (p.pool_mode[li] == 0) {
      DevBuf out;
      float* dst = last ? final_slot() : nullptr;
      if (!last) {
        out.alloc(m.c, B * entry_bytes(so));
        dst = out.as<float>();
      }
      const int h = timer.begin(li);
      launch_maxpool(m.c, in, B, si.f, si.n, l.ext, dst);
      timer.end(h);
      if (owner) owner->reset();
      if (last) {
        final_off += B;
        return;
      }
      run(li + 1, dst, &out, B);
      return;
    }
    const int64_t total = B * l.ext.vol();
    int64_t G = total;
    if (!last) {
      PeakModel pm{m, p, cache};
      int64_t avail;
      {
        std::lock_guard<std::mutex> lk(m.c->mu);
        avail = m.c->budget - m.c->current;
      }
      G = pm.choose(li, B, avail + B * entry_bytes(si));
    }
    for (int64_t b0 = 0; b0 < total; b0 += G) {
      const int64_t g = std::min(G, total - b0);
      DevBuf out;
      float* dst = last ? final_slot() : nullptr;
      if (!last) {
        out.alloc(m.c, g * entry_bytes(so));
        dst = out.as<float>();
      }
      const int h = timer.begin(li);
      launch_mpf(m.c, in, B, si.f, si.n, l.ext, dst, b0, g);
      timer.end(h);
      if (last) {
        final_off += g;
        continue;
      }
      run(li + 1, dst, &out, g);
    }
    if (owner) owner->reset();
  }
};

}  // namespace

const float2* Model::spectra_for(int ci, int T, bool cache) {
  if (!cache) return nullptr;
  auto key = std::make_pair(ci, T);
  auto it = spectra.find(key);
  if (it != spectra.end()) return it->second.as<float2>();
  // locate the layer of conv ordinal ci
  int64_t f = net.fin;
  for (size_t li = 0; li < net.layers.size(); ++li) {
    const Layer& l = net.layers[li];
    if (l.kind != 0) continue;
    if (conv_index[li] == ci) {
      DevBuf b(c, tile_nwb(T) * l.fo * f * 16 * 8);
      compute_kernel_spectra(c, T, kern[size_t(ci)].as<float>(), l.fo, f, l.ext, b.as<float2>());
      auto res = spectra.emplace(key, std::move(b));
      return res.first->second.as<float2>();
    }
    f = l.fo;
  }
  throw invalid("model: unknown conv layer");
}

int64_t Model::plan_bytes(const ForwardPlan& p, bool cache) const {
  PeakModel pm{*this, p, cache};
  const int64_t in = p.S * entry_bytes(p.shapes[0]);
  const int64_t frags = p.S * p.alpha * entry_bytes(p.shapes.back());
  const int64_t dense = p.S * p.f_out * p.dense.vol() * 4;
  int64_t spectra_bytes = 0;
  if (cache) {
    int64_t f = net.fin;
    for (size_t li = 0; li < net.layers.size(); ++li) {
      const Layer& l = net.layers[li];
      if (l.kind != 0) continue;
      if (p.choice[li].algo == VXG_CONV_FFT) spectra_bytes += p.choice[li].fft.nwb * l.fo * f * 128;
      f = l.fo;
    }
  }
  // smallest groups: the feasibility threshold
  const int64_t huge = int64_t(1) << 62;
  (void)huge;
  int64_t minimal = 0;
  {
    // peak with avail = 0 forces g = 1 at every pool
    minimal = pm.peak(0, p.S, 0);
  }
  return minimal + frags + dense + spectra_bytes + (in - p.S * entry_bytes(p.shapes[0]));
}

void Model::forward(const ForwardPlan& p, const float* d_in, float* d_dense, bool cache,
                    std::vector<double>* layer_seconds) {
  EventTimer timer(c->stream, layer_seconds != nullptr);
  DevBuf frags(c, p.S * p.alpha * entry_bytes(p.shapes.back()));
  Runner r{*this, p, cache, frags.as<float>(), 0, timer};
  r.run(0, d_in, nullptr, p.S);
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
