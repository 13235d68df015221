// Network grammar, shape rules and synthetic data (see net.hpp for the
// reference interfaces each function replaces).
#include "net.hpp"

#include <cmath>
#include <random>
#include <sstream>

namespace vxg {

i64 Net::conv_count() const {
  i64 c = 0;
  for (const auto& l : layers) c += l.kind == 0;
  return c;
}
i64 Net::pool_count() const { return i64(layers.size()) - conv_count(); }
i64 Net::features_out() const {
  i64 f = fin;
  for (const auto& l : layers)
    if (l.kind == 0) f = l.fo;
  return f;
}

// NetworkSpec::validate (network.hpp:52-64)
void Net::validate() const {
  require(fin > 0, "NetworkSpec: features_in must be positive");
  require(!layers.empty(), "NetworkSpec: at least one layer required");
  for (const auto& l : layers) {
    if (l.kind == 0) {
      require(l.fo > 0, "NetworkSpec: conv features_out must be positive");
      require(l.ext.positive(), "NetworkSpec: conv kernel extents must be positive");
    } else {
      require(l.ext.positive(), "NetworkSpec: pool window extents must be positive");
    }
  }
}

i64 Net::weight_count() const {
  i64 f = fin, total = 0;
  for (const auto& l : layers)
    if (l.kind == 0) {
      total += l.fo * f * l.ext.vol() + l.fo;
      f = l.fo;
    }
  return total;
}

namespace {

[[noreturn]] void perr(i64 line, const std::string& msg) {
  throw parse_failure("line " + std::to_string(line) + ": " + msg);
}

std::vector<std::string> tokens_of(std::string line) {
  const auto hash = line.find('#');
  if (hash != std::string::npos) line.erase(hash);
  std::vector<std::string> t;
  std::istringstream ss(line);
  std::string w;
  while (ss >> w) t.push_back(w);
  return t;
}

i64 number_of(const std::string& tok, i64 line) {
  size_t pos = 0;
  long long v = 0;
  bool ok = true;
  try {
    v = std::stoll(tok, &pos);
  } catch (...) {
    ok = false;
  }
  if (!ok || pos != tok.size()) perr(line, "expected a number, got '" + tok + "'");
  return v;
}

i64 extent_of(const std::string& tok, i64 line) {
  const i64 v = number_of(tok, line);
  if (v < 1) perr(line, "extent must be >= 1");
  return v;
}

V3 extents_of(const std::vector<std::string>& t, size_t first, size_t count, i64 line,
              const char* what) {
  if (count == 1) return V3::cube(extent_of(t[first], line));
  if (count == 3)
    return V3{extent_of(t[first], line), extent_of(t[first + 1], line),
              extent_of(t[first + 2], line)};
  perr(line, what);
}

}  // namespace

// parse_network_spec (netspec.cpp:54-120): same grammar, same diagnostics.
Net parse_net(const std::string& text) {
  Net net;
  bool saw_input = false;
  i64 line_no = 0;
  std::istringstream lines(text);
  std::string line;
  while (std::getline(lines, line)) {
    ++line_no;
    const auto t = tokens_of(line);
    if (t.empty()) continue;
    const std::string& kw = t[0];
    if (kw == "input") {
      if (saw_input) perr(line_no, "duplicate input declaration");
      if (!net.layers.empty()) perr(line_no, "input must precede the layers");
      if (t.size() != 2) perr(line_no, "input takes one feature count");
      net.fin = number_of(t[1], line_no);
      if (net.fin < 1) perr(line_no, "feature count must be >= 1");
      saw_input = true;
      continue;
    }
    if (!saw_input) perr(line_no, "missing input declaration");
    if (kw == "conv") {
      size_t n = t.size() - 1;
      bool relu = false;
      if (n >= 1 && t.back() == "relu") {
        relu = true;
        --n;
      }
      if (n != 2 && n != 4) perr(line_no, "conv takes a feature count and one or three kernel extents");
      const i64 fo = number_of(t[1], line_no);
      if (fo < 1) perr(line_no, "feature count must be >= 1");
      Layer l;
      l.kind = 0;
      l.fo = fo;
      l.relu = relu;
      l.ext = extents_of(t, 2, n - 1, line_no,
                         "conv takes a feature count and one or three kernel extents");
      net.layers.push_back(l);
      continue;
    }
    if (kw == "pool") {
      size_t n = t.size() - 1;
      int mode = -1;
      if (n >= 1) {
        const std::string& last = t.back();
        if (last == "mpf" || last == "plain" || last == "auto") {
          if (last == "mpf") mode = 1;
          if (last == "plain") mode = 0;
          --n;
        }
      }
      Layer l;
      l.kind = 1;
      l.forced = mode;
      l.ext = extents_of(t, 1, n, line_no, "pool takes one or three window extents");
      net.layers.push_back(l);
      continue;
    }
    perr(line_no, "unknown keyword '" + kw + "'");
  }
  if (!saw_input) perr(line_no > 1 ? line_no : 1, "missing input declaration");
  if (net.layers.empty()) perr(line_no > 1 ? line_no : 1, "network needs at least one layer");
  net.validate();
  return net;
}

// format_network_spec (netspec.cpp:133-151)
std::string format_net(const Net& net) {
  std::ostringstream out;
  auto put = [&](const V3& v) {
    if (v.x == v.y && v.y == v.z)
      out << v.x;
    else
      out << v.x << ' ' << v.y << ' ' << v.z;
  };
  out << "input " << net.fin << '\n';
  for (const auto& l : net.layers) {
    if (l.kind == 0) {
      out << "conv " << l.fo << ' ';
      put(l.ext);
      if (l.relu) out << " relu";
    } else {
      out << "pool ";
      put(l.ext);
      if (l.forced >= 0) out << (l.forced == 1 ? " mpf" : " plain");
    }
    out << '\n';
  }
  return out.str();
}

// field_of_view (cost.cpp:107-122): fov += (k-1)*stride; pools also grow stride
V3 field_of_view(const Net& net) {
  net.validate();
  V3 fov{1, 1, 1}, stride{1, 1, 1};
  for (const auto& l : net.layers)
    for (int a = 0; a < 3; ++a) {
      fov[a] += (l.ext[a] - 1) * stride[a];
      if (l.kind == 1) stride[a] *= l.ext[a];
    }
  return fov;
}

// propagate_shapes (planner.cpp:536-589)
std::vector<Shape> propagate_shapes(const Net& net, Shape cur, const std::vector<int>& modes_in,
                                    i64* violation) {
  net.validate();
  require(cur.s > 0 && cur.f > 0 && cur.n.positive(), "Shape5: all extents must be positive");
  require(cur.f == net.fin, "propagate_shapes: input features must match the network");
  std::vector<int> modes = modes_in;
  if (modes.empty()) modes.assign(size_t(net.pool_count()), 1);
  require(i64(modes.size()) == net.pool_count(),
          "propagate_shapes: one mode per pooling layer required");
  std::vector<Shape> chain{cur};
  *violation = -1;
  size_t pi = 0;
  for (i64 li = 0; li < i64(net.layers.size()); ++li) {
    const Layer& l = net.layers[size_t(li)];
    if (l.kind == 0) {
      for (int a = 0; a < 3; ++a)
        if (cur.n[a] < l.ext[a]) {
          *violation = li;
          return chain;
        }
      for (int a = 0; a < 3; ++a) cur.n[a] = cur.n[a] - l.ext[a] + 1;
      cur.f = l.fo;
    } else {
      const int mode = modes[pi++];
      if (l.forced >= 0)
        require(l.forced == mode, "propagate_shapes: assignment conflicts with a forced pooling mode");
      for (int a = 0; a < 3; ++a) {
        const bool bad = mode == 0 ? cur.n[a] % l.ext[a] != 0 : (cur.n[a] + 1) % l.ext[a] != 0;
        if (bad) {
          *violation = li;
          return chain;
        }
      }
      for (int a = 0; a < 3; ++a) cur.n[a] = cur.n[a] / l.ext[a];
      if (mode == 1) cur.s *= l.ext.vol();
    }
    chain.push_back(cur);
  }
  return chain;
}

// random_weights (execute.hpp:50-73): one mt19937_64 stream; per conv layer
// all kernel entries U(+-sqrt(3/(f*k^3))) then biases U(+-0.1).
void random_weights(const Net& net, uint64_t seed, float* out) {
  net.validate();
  std::mt19937_64 rng(seed);
  i64 f = net.fin, off = 0;
  for (const auto& l : net.layers) {
    if (l.kind != 0) continue;
    const double bound = std::sqrt(3.0 / (double(f) * double(l.ext.vol())));
    std::uniform_real_distribution<double> kd(-bound, bound);
    std::uniform_real_distribution<double> bd(-0.1, 0.1);
    const i64 nk = l.fo * f * l.ext.vol();
    for (i64 i = 0; i < nk; ++i) out[off++] = float(kd(rng));
    for (i64 i = 0; i < l.fo; ++i) out[off++] = float(bd(rng));
    f = l.fo;
  }
}

// fill_random (cli.cpp:78-84)
void fill_random(float* out, i64 count, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> d(-1.0, 1.0);
  for (i64 i = 0; i < count; ++i) out[i] = float(d(rng));
}

}  // namespace vxg
