// Shared host/device plumbing of the vxg library: error types that map onto
// the C-ABI status codes, the per-GPU context (stream + budgeted
// stream-ordered allocator = the device MemoryTracker of
// proj/include/voxin/memory.hpp:15-51 with byte units), and launch helpers.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <map>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "vxg.h"

namespace vxg {

using i64 = int64_t;

struct invalid : std::invalid_argument {
  explicit invalid(const std::string& w) : std::invalid_argument(w) {}
};
struct exhausted : std::runtime_error {
  explicit exhausted(const std::string& w) : std::runtime_error(w) {}
};
struct cuda_failure : std::runtime_error {
  explicit cuda_failure(const std::string& w) : std::runtime_error(w) {}
};
struct parse_failure : std::runtime_error {
  explicit parse_failure(const std::string& w) : std::runtime_error(w) {}
};

// VXG_TRACE=1: the executor and layer drivers print their plans to stderr
bool trace_on();

inline void require(bool cond, const char* what) {
  if (!cond) throw invalid(what);
}

#define VXG_CUDA_CHECK(expr)                                                             \
  do {                                                                                   \
    cudaError_t e__ = (expr);                                                            \
    if (e__ != cudaSuccess)                                                              \
      throw ::vxg::cuda_failure(std::string(#expr) + ": " + cudaGetErrorString(e__));    \
  } while (0)

struct V3 {
  i64 x = 1, y = 1, z = 1;
  i64 operator[](int a) const { return a == 0 ? x : (a == 1 ? y : z); }
  i64& operator[](int a) { return a == 0 ? x : (a == 1 ? y : z); }
  i64 vol() const { return x * y * z; }
  bool positive() const { return x > 0 && y > 0 && z > 0; }
  bool operator==(const V3& o) const { return x == o.x && y == o.y && z == o.z; }
  static V3 of(const int64_t* a) { return V3{a[0], a[1], a[2]}; }
  static V3 cube(i64 e) { return V3{e, e, e}; }
};

// Per-launch instrumentation record (CUDA events on the launching stream plus
// the launch's ALGORITHMIC flops / bytes), enabled by vxg_ctx_profile().
struct KRecord {
  int kind;
  cudaEvent_t a, b;
  double flops, bytes;
};

// Best-fit sub-allocator over one device block (coalescing free list).  All
// work runs on the context's single stream, so a block freed on the host may
// be handed out again at once: the next user is stream-ordered after the last.
struct Arena {
  char* base = nullptr;
  i64 size = 0;
  std::map<i64, i64> free_;  // offset -> bytes

  i64 used = 0, peak = 0;    // bytes handed out now / at most (the forward's audit)

  static constexpr i64 kAlign = 512;
  void reset(void* b, i64 n) {
    base = static_cast<char*>(b);
    size = n;
    used = peak = 0;
    free_.clear();
    if (n > 0) free_[0] = n;
  }
  void* alloc(i64 bytes) {
    bytes = (bytes + kAlign - 1) / kAlign * kAlign;
    auto best = free_.end();
    for (auto it = free_.begin(); it != free_.end(); ++it)
      if (it->second >= bytes && (best == free_.end() || it->second < best->second)) best = it;
    if (best == free_.end()) return nullptr;
    const i64 off = best->first, len = best->second;
    free_.erase(best);
    if (len > bytes) free_[off + bytes] = len - bytes;
    used += bytes;
    if (used > peak) peak = used;
    return base + off;
  }
  void release(void* p, i64 bytes) {
    bytes = (bytes + kAlign - 1) / kAlign * kAlign;
    used -= bytes;
    i64 off = static_cast<char*>(p) - base;
    auto next = free_.lower_bound(off);
    if (next != free_.end() && next->first == off + bytes) {
      bytes += next->second;
      next = free_.erase(next);
    }
    if (next != free_.begin()) {
      auto prev = std::prev(next);
      if (prev->first + prev->second == off) {
        prev->second += bytes;
        return;
      }
    }
    free_[off] = bytes;
  }
  bool owns(const void* p) const {
    const char* q = static_cast<const char*>(p);
    return base && q >= base && q < base + size;
  }
  i64 largest() const {
    i64 m = 0;
    for (const auto& kv : free_) m = std::max(m, kv.second);
    return m;
  }
};

// One-time setup per device (kernel attributes such as the dynamic shared
// memory limit are per device): first() is true once for each device.
struct PerDeviceOnce {
  std::atomic<unsigned long long> mask{0};
  bool first() {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long b = 1ull << (d & 63);
    return !(mask.fetch_or(b) & b);
  }
};

// One context per GPU.  All work is issued on `stream`; allocations are
// stream-ordered (cudaMallocAsync) and charged against `budget` bytes.
struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaMemPool_t pool = nullptr;
  i64 budget = 0;
  i64 current = 0;
  i64 peak = 0;
  int num_sms = 148;
  int* d_flag = nullptr;  // device error flag (NaN seen by pools)
  std::atomic<i64> launches{0};
  std::mutex mu;
  bool prof = false;
  std::vector<KRecord> krec;
  std::vector<cudaEvent_t> spare_events;
  Arena* arena = nullptr;  // set while a network forward runs (forward.cu)
  // the forward's arena block, kept between forwards (a freed block of that
  // size is split by the pool for the next forward's smaller requests, after
  // which the arena no longer fits and the pool trims and remaps ~100 GB);
  // charged against the budget only while a forward uses it, and handed back
  // to the pool whenever a device allocation would not fit without it
  void* held = nullptr;
  i64 held_bytes = 0;
  bool held_busy = false;

  // device bytes really obtainable now: free memory plus what the pool holds
  // unused (other users of the GPU -- e.g. torch tensors allocated after the
  // budget was set -- are not in the budget)
  i64 device_free() {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return budget;
    unsigned long long reserved = 0, used = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    return i64(fr) + i64(reserved) - i64(used);
  }

  // bytes a new allocation can get: the largest arena block, else the budget left
  i64 avail() {
    std::lock_guard<std::mutex> lk(mu);
    return arena ? arena->largest() : budget - current;
  }

  cudaEvent_t take_event() {
    if (!spare_events.empty()) {
      cudaEvent_t e = spare_events.back();
      spare_events.pop_back();
      return e;
    }
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) throw cuda_failure("cudaEventCreate failed");
    return e;
  }

  void charge(i64 bytes) {
    std::lock_guard<std::mutex> lk(mu);
    if (current + bytes > budget)
      throw exhausted("HBM budget exceeded: need " + std::to_string(current + bytes) +
                      " bytes, budget " + std::to_string(budget));
    current += bytes;
    if (current > peak) peak = current;
  }
  void release(i64 bytes) {
    std::lock_guard<std::mutex> lk(mu);
    current -= bytes;
  }
  void counted(i64 n = 1) { launches += n; }
  // give the held arena block back to the pool (not while a forward uses it)
  bool drop_held() {
    void* p = nullptr;
    {
      std::lock_guard<std::mutex> lk(mu);  // another context's thread may call this (release_idle_memory)
      if (!held || held_busy) return false;
      p = held;
      held = nullptr;
      held_bytes = 0;
    }
    cudaFreeAsync(p, stream);
    return true;
  }
};

// Contexts of this process (api.cu).  release_idle_memory hands the idle
// cached device memory of every context on `device` -- held arena blocks and
// the pools' unused reserves -- back to the driver: caches yield to any
// allocation that would otherwise fail (another context's, or this one's).
void register_ctx(Ctx* c);
void unregister_ctx(Ctx* c);
void release_idle_memory(int device);

// Brackets one kernel launch with events when profiling is on.
class KScope {
 public:
  KScope(Ctx* c, int kind, double flops, double bytes) : c_(c) {
    if (!c_->prof) return;
    rec_ = KRecord{kind, c_->take_event(), c_->take_event(), flops, bytes};
    cudaEventRecord(rec_.a, c_->stream);
  }
  ~KScope() {
    if (!c_->prof) return;
    cudaEventRecord(rec_.b, c_->stream);
    c_->krec.push_back(rec_);
  }
  KScope(const KScope&) = delete;
  KScope& operator=(const KScope&) = delete;

 private:
  Ctx* c_;
  KRecord rec_{};
};

// RAII device buffer charged against the context budget.
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(Ctx* c, i64 bytes) { alloc(c, bytes); }
  ~DevBuf() { reset(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : c_(o.c_), p_(o.p_), n_(o.n_), arena_(o.arena_) {
    o.c_ = nullptr; o.p_ = nullptr; o.n_ = 0; o.arena_ = nullptr;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      c_ = o.c_; p_ = o.p_; n_ = o.n_; arena_ = o.arena_;
      o.c_ = nullptr; o.p_ = nullptr; o.n_ = 0; o.arena_ = nullptr;
    }
    return *this;
  }
  void alloc(Ctx* c, i64 bytes) {
    reset();
    if (bytes <= 0) return;
    i64 arena_largest = -1;
    if (c->arena) {
      void* q = nullptr;
      Arena* ar = nullptr;
      {
        std::lock_guard<std::mutex> lk(c->mu);
        ar = c->arena;
        if (ar) {
          q = ar->alloc(bytes);
          if (!q) arena_largest = ar->largest();
        }
      }
      if (q) {
        c_ = c; p_ = q; n_ = bytes; arena_ = ar;
        return;
      }
    }
    c->charge(bytes);
    void* p = nullptr;
    if (trace_on() && arena_largest >= 0)
      std::fprintf(stderr, "[vxg] arena miss: %lld bytes from the pool (arena largest free %lld)\n",
                   (long long)bytes, (long long)arena_largest);
    cudaError_t e = cudaMallocFromPoolAsync(&p, static_cast<size_t>(bytes), c->pool, c->stream);
    if (e == cudaErrorMemoryAllocation) {
      if (trace_on()) std::fprintf(stderr, "[vxg] pool trim + remap for %lld bytes\n", (long long)bytes);
      // the pool keeps freed blocks mapped (release threshold = max); when none
      // of them fits, hand them back and map the request afresh
      cudaGetLastError();
      release_idle_memory(c->device);
      cudaStreamSynchronize(c->stream);
      cudaMemPoolTrimTo(c->pool, 0);
      e = cudaMallocFromPoolAsync(&p, static_cast<size_t>(bytes), c->pool, c->stream);
    }
    if (e != cudaSuccess) {
      c->release(bytes);
      cudaGetLastError();
      if (e == cudaErrorMemoryAllocation)
        throw exhausted("device allocation of " + std::to_string(bytes) + " bytes failed");
      throw cuda_failure(std::string("cudaMallocFromPoolAsync: ") + cudaGetErrorString(e));
    }
    c_ = c; p_ = p; n_ = bytes;
  }
  void reset() {
    if (p_ && arena_) {
      std::lock_guard<std::mutex> lk(c_->mu);
      arena_->release(p_, n_);
    } else if (p_) {
      cudaFreeAsync(p_, c_->stream);
      c_->release(n_);
    }
    c_ = nullptr; p_ = nullptr; n_ = 0; arena_ = nullptr;
  }
  template <class T = float>
  T* as() const { return static_cast<T*>(p_); }
  void* get() const { return p_; }
  // detach a pool allocation (the caller keeps it, and its budget charge)
  void* release_ptr() {
    void* q = p_;
    p_ = nullptr;
    n_ = 0;
    c_ = nullptr;
    return q;
  }
  i64 bytes() const { return n_; }

 private:
  Ctx* c_ = nullptr;
  void* p_ = nullptr;
  i64 n_ = 0;
  Arena* arena_ = nullptr;
};

inline unsigned grid_for(i64 n, int block, i64 cap = (i64(1) << 31) - 1) {
  i64 g = (n + block - 1) / block;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw cuda_failure(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- kernel entry points (implemented in the k_*.cu units) -----------------

// pools (k_pool.cu)
// MPF of S whole entries (all P fragments); the output may be the channel
// slice [c0, c0+f) of a tensor with f_tot channels (f_tot <= 0: f)
// ipz / opz: z row pitch of input / output (0: unpadded)
// mx_out / x_out0: the pooled fragments of an x slab of the input go to x
// positions [x_out0, x_out0 + n.x / 2) of fragments mx_out wide (2x2x2 only)
void launch_mpf(Ctx* c, const float* in, i64 S, i64 f, V3 n, V3 p, float* out, i64 f_tot = 0,
                i64 c0 = 0, i64 ipz = 0, i64 opz = 0, i64 mx_out = 0, i64 x_out0 = 0);
void launch_maxpool(Ctx* c, const float* in, i64 S, i64 f, V3 n, V3 p, float* out);
void launch_recombine(Ctx* c, const float* frag, i64 nfrag, i64 b0, i64 f, V3 n,
                      const i64* windows, int nwin, float* dense, i64 S0, i64 fpz = 0);
void launch_nan_check(Ctx* c, const float* x, i64 count);
bool read_and_clear_flag(Ctx* c);
void clear_flag_async(Ctx* c);

// instrumentation (k_misc.cu)
double bench_ffma(Ctx* c);

// direct convolution (k_direct.cu)
void launch_conv_direct(Ctx* c, const float* in, i64 S, i64 f, V3 n, const float* w, i64 fo,
                        V3 k, const float* bias, bool relu, float* out, i64 ipz = 0, i64 opz = 0);
// f = 1 direct convolution on the tensor cores (k_direct_tc.cu); VXG_DIRECT_TC=0 disables
bool direct_tc_supported(int64_t f, int64_t fo, V3 k, const void* in);
void launch_direct_tc(Ctx* c, const float* in, i64 S, V3 n, const float* w, i64 fo, V3 k, const float* bias,
                      bool relu, float* out, i64 ipz, i64 opz);

}  // namespace vxg
