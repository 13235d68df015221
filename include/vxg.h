/* vxg — B200-native sliding-window 3D ConvNet inference (ZNNi hot path).
 *
 * The drop-in C-ABI boundary.  Plain pointers and int64 sizes only; every
 * function returns a status code (VXG_OK = 0) and leaves a thread-local
 * message in vxg_last_error().  Tensors are fp32, row-major in the
 * reference's Tensor5 layout (s, f, x, y, z), z fastest
 * (proj/include/voxin/shape.hpp:31-33).  `mem` selects whether tensor
 * pointers are host memory (copied in and out inside the call, which is then
 * synchronous) or device memory (the call is stream-ordered on the context's
 * stream; vxg_ctx_sync() waits).
 *
 * Each entry point replaces one reference interface (paths relative to
 * /root/reference/proj); the status codes map onto the reference's error
 * conventions: VXG_INVALID <-> std::invalid_argument via require()
 * (include/voxin/common.hpp:16-18), VXG_EXHAUSTED <-> vx::resource_exhausted
 * (common.hpp:12-14), VXG_PARSE <-> vx::ParseError (netspec.hpp:11-20).
 */
#ifndef VXG_H_
#define VXG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum vxg_status {
  VXG_OK = 0,
  VXG_INVALID = 1,   /* std::invalid_argument: shape / contract violation */
  VXG_EXHAUSTED = 2, /* vx::resource_exhausted: HBM budget or workspace cap */
  VXG_CUDA = 3,      /* CUDA runtime error (no CPU fallback exists) */
  VXG_PARSE = 4,     /* vx::ParseError: malformed network text (message has the line) */
  VXG_INTERNAL = 5
};

enum vxg_mem { VXG_MEM_HOST = 0, VXG_MEM_DEVICE = 1 };

/* Convolution algorithms (the PrimitiveKind conv kinds of
 * include/voxin/cost.hpp:13-24 collapse to these two device algorithms). */
enum vxg_conv_algo {
  VXG_CONV_AUTO = 0,   /* planner's choice (cost model) */
  VXG_CONV_DIRECT = 1, /* conv_direct (layers.hpp:142-192) */
  VXG_CONV_FFT = 2     /* conv_fft_{data_parallel,staged,task_parallel} (layers.hpp:203-371,
                          task_conv.hpp:415-442): tiled pruned-FFT convolution */
};

/* FFT radix profiles of RadixProfile (include/voxin/fft.hpp:17-47). */
enum vxg_profile { VXG_PROFILE_HOST = 0, VXG_PROFILE_DEVICE = 1, VXG_PROFILE_ANY = 2 };

/* vx::MemoryAudit (include/voxin/memory.hpp:100-103): real-scalar units. */
typedef struct {
  double peak;  /* device allocator high-water mark of the call, scalars (bytes / 4) */
  double model; /* closed-form working-set model of the algorithm used, scalars */
} vxg_audit;

/* vx::ThroughputReport (include/voxin/execute.hpp:76-84), device flavour. */
typedef struct {
  double voxels;            /* recombined dense output voxels, batch included */
  double seconds;           /* device time of the forward (CUDA events) */
  double voxels_per_second;
  double device_peak;       /* audited peak working set, scalars */
  int64_t layers;           /* entries written to layer_seconds */
  double layer_seconds[64]; /* per network layer, device time */
} vxg_report;

typedef struct vxg_ctx vxg_ctx;
typedef struct vxg_net vxg_net;

const char* vxg_last_error(void);
const char* vxg_version(void);

/* ---- context: one per GPU, one host thread per context ------------------- */
/* The context owns a CUDA stream, a stream-ordered allocator and the HBM budget
 * tracker (the device MemoryTracker of execute.hpp:259-267).  budget <= 0:
 * the free HBM at creation minus a 2.5 GiB reserve. */
int vxg_ctx_create(int device, int64_t hbm_budget_bytes, vxg_ctx** out);
int vxg_ctx_destroy(vxg_ctx* ctx);
int vxg_ctx_sync(vxg_ctx* ctx);
int vxg_ctx_stream(vxg_ctx* ctx, void** cuda_stream);
/* bytes currently held / high-water mark since the last reset */
int vxg_ctx_memory(vxg_ctx* ctx, int64_t* current, int64_t* peak, int64_t* budget);
/* Hand the network forward's cached arena block back to the device pool (it
 * is kept between forwards so the next forward reuses it without remapping;
 * the library drops it by itself when another allocation would not fit).
 * No reference counterpart (the reference's host arenas are per call). */
int vxg_ctx_trim(vxg_ctx* ctx);
int vxg_ctx_reset_peak(vxg_ctx* ctx);
/* number of kernels this context launched so far (for launch accounting) */
int64_t vxg_ctx_launches(vxg_ctx* ctx);

/* Kernel families for per-launch instrumentation. */
enum vxg_kernel_kind {
  VXG_K_TILE_FWD = 0, /* K1: forward tile transform (images) */
  VXG_K_TILE_INV = 1, /* K4: inverse tile transform + crop/bias/ReLU */
  VXG_K_CGEMM = 2,    /* K3: per-frequency complex contraction */
  VXG_K_KSPEC = 3,    /* K2: kernel spectra */
  VXG_K_DIRECT = 4,   /* K5: direct convolution */
  VXG_K_POOL = 5,     /* K6: MPF / max pooling */
  VXG_K_RECOMBINE = 6,/* K7: fragment recombination */
  VXG_K_LINEFFT = 7,  /* whole-image transform lines */
  VXG_K_OTHER = 8,
  VXG_K_COUNT = 9
};
/* enable != 0: start recording CUDA events around every launch (clears old
 * records); 0: stop. */
int vxg_ctx_profile(vxg_ctx* ctx, int enable);
/* Aggregate of the recorded launches of one kind: count, summed device
 * seconds, summed algorithmic flops and bytes (synchronises the stream). */
int vxg_ctx_kernel_stats(vxg_ctx* ctx, int kind, int64_t* launches, double* seconds,
                         double* flops, double* bytes);
/* FFMA throughput microbenchmark (TFLOP/s, fp32, all SMs): the roofline
 * denominator of the FFMA kernels (MEASURED_PEAKS.json has no fp32 figure). */
int vxg_bench_ffma(vxg_ctx* ctx, double* tflops);

/* ---- layer primitives (include/voxin/layers.hpp) -------------------------- */

/* conv_direct / conv_fft_* (layers.hpp:142-371, task_conv.hpp:415-442):
 *   out(S, fo, n-k+1) = act(bias + sum_i kernels(fo, f, k) (*) in(S, f, n))
 * valid TRUE convolution (kernel index-reversed), relu != 0 -> ReLU. */
int vxg_conv(vxg_ctx* ctx, int algo, int mem, const float* in, int64_t S, int64_t f,
             const int64_t n[3], const float* kernels, int64_t fo, const int64_t k[3],
             const float* bias, int relu, float* out, vxg_audit* audit);

/* The FFT convolution of vxg_conv with the plan pinned by the caller (parity
 * tests, experiments): tile FFT size `tile` (must cover the kernel; one of
 * 4 6 8 10 12 16 20 24 28 30 32), flags VXG_FFT_FFMA (fp32 FFMA contraction
 * instead of tcgen05), VXG_FFT_SINGLE_CTA (no CTA-pair forward transform);
 * spectra_budget > 0 caps the spectrum chunk buffers (bytes), forcing the
 * multi-chunk path. */
#define VXG_FFT_FFMA 1
#define VXG_FFT_SINGLE_CTA 2
int vxg_conv_fft_tiled(vxg_ctx* ctx, int mem, const float* in, int64_t S, int64_t f,
                       const int64_t n[3], const float* kernels, int64_t fo, const int64_t k[3],
                       const float* bias, int relu, float* out, int tile, int flags,
                       int64_t spectra_budget);

/* max_pool (layers.hpp:377-417): n % p == 0; NaN input -> VXG_INVALID. */
int vxg_max_pool(vxg_ctx* ctx, int mem, const float* in, int64_t S, int64_t f,
                 const int64_t n[3], const int64_t p[3], float* out, vxg_audit* audit);

/* mpf_pool (layers.hpp:424-470): (n+1) % p == 0; out (S*P, f, floor(n/p)),
 * batch index s*P + (ox*py*pz + oy*pz + oz).  Bit-exact. */
int vxg_mpf_pool(vxg_ctx* ctx, int mem, const float* in, int64_t S, int64_t f,
                 const int64_t n[3], const int64_t p[3], float* out, vxg_audit* audit);

/* recombine_fragments (layers.hpp:477-520): windows is nwin x 3 (network
 * order); frag batch = original_batch * prod(|windows|).  Bit-exact. */
int vxg_recombine(vxg_ctx* ctx, int mem, const float* frag, int64_t S_frag, int64_t f,
                  const int64_t n[3], const int64_t* windows, int64_t nwin,
                  int64_t original_batch, float* dense);

/* ---- transforms (include/voxin/fft.hpp:392-457) ----------------------------- */

/* optimal_fft_size (fft.hpp:50-56) */
int64_t vxg_optimal_fft_size(int64_t n, int profile);

/* pruned_fft_forward: spec = (floor(pad_x/2)+1, pad_y, pad_z) complex64, interleaved */
int vxg_fft_pruned_forward(vxg_ctx* ctx, int mem, const float* img, const int64_t n[3],
                           const int64_t pad[3], float* spec);
/* pruned_fft_inverse: low-corner crop, scaled by 1/(pad_x*pad_y*pad_z) */
int vxg_fft_pruned_inverse(vxg_ctx* ctx, int mem, const float* spec, const int64_t pad[3],
                           const int64_t crop[3], float* out);
/* batched_fft_forward: spec = (b, floor(pad_z/2)+1, pad_y, pad_x) complex64 */
int vxg_fft_batched_forward(vxg_ctx* ctx, int mem, const float* imgs, int64_t b,
                            const int64_t n[3], const int64_t pad[3], float* spec);
/* batched_fft_inverse: (b, crop) */
int vxg_fft_batched_inverse(vxg_ctx* ctx, int mem, const float* spec, int64_t b,
                            const int64_t pad[3], const int64_t crop[3], float* out);

/* ---- network description (include/voxin/network.hpp, netspec.hpp) ---------- */

/* parse_network_spec (src/netspec.cpp:54-120); VXG_PARSE with "line N: ..." */
int vxg_net_parse(const char* text, vxg_net** out);
int vxg_net_free(vxg_net* net);
/* format_network_spec (netspec.cpp:133-151); writes at most cap bytes (NUL incl.);
 * *needed = bytes required */
int vxg_net_format(const vxg_net* net, char* buf, int64_t cap, int64_t* needed);
/* layer count, conv count, pool count, input features, output features */
int vxg_net_info(const vxg_net* net, int64_t info[5]);
/* layer l: kind (0 conv, 1 pool), extents (kernel / window), features_out (conv),
 * relu (conv), forced pool mode (-1 auto, 0 plain, 1 fragments) */
int vxg_net_layer(const vxg_net* net, int64_t l, int64_t* kind, int64_t ext[3], int64_t* fo,
                  int64_t* relu, int64_t* forced_mode);
/* field_of_view (src/cost.cpp:107-122) */
int vxg_net_fov(const vxg_net* net, int64_t fov[3]);
/* propagate_shapes (src/planner.cpp:536-589): pool_modes one per pool (0 plain,
 * 1 fragments) or NULL for all-fragments; shapes receives (layers+1) x 5
 * (s, f, x, y, z); *violation = offending layer or -1. */
int vxg_net_propagate(const vxg_net* net, int64_t S, const int64_t e[3], const int* pool_modes,
                      int64_t* shapes, int64_t* violation);
/* total weight scalars: per conv layer kernels (fo, f, k) then biases (fo) */
int64_t vxg_net_weight_count(const vxg_net* net);
/* random_weights (include/voxin/execute.hpp:50-73), flat in the order above */
int vxg_random_weights(const vxg_net* net, uint64_t seed, float* weights);
/* fill_random (src/cli.cpp:78-84): mt19937_64(seed), U(-1, 1) */
int vxg_fill_random(float* out, int64_t count, uint64_t seed);

/* ---- network forward (include/voxin/execute.hpp:388-402) --------------------- */

/* Dense sliding-window inference of `net` over input (S, f_in, e): every pool
 * runs as MPF, fragments recombined (execute_plan with an all-fragment plan).
 * weights as vxg_random_weights.  conv_algos: one vxg_conv_algo per conv layer,
 * or NULL for the planner's choice.  dense_out: (S, f_out, e - fov + 1).
 * Activations stay device-resident; fragment sub-batches bound HBM use. */
int vxg_net_forward(vxg_ctx* ctx, const vxg_net* net, const float* weights, int mem,
                    const float* input, int64_t S, const int64_t e[3], const int* conv_algos,
                    float* dense_out, vxg_report* report);

/* Device-resident weights for repeated forwards (kernel spectra cached per
 * layer and FFT tile size, the "kernel-spectrum cache" of SURVEY 8f).
 * weights == NULL creates a planning-only model (plan queries only). */
typedef struct vxg_model vxg_model;
int vxg_model_create(vxg_ctx* ctx, const vxg_net* net, const float* weights, int mem,
                     vxg_model** out);
int vxg_model_free(vxg_model* model);
/* cache_spectra = 0: kernel spectra are recomputed inside every forward */
int vxg_model_forward(vxg_model* model, int mem, const float* input, int64_t S,
                      const int64_t e[3], const int* conv_algos, int cache_spectra,
                      float* dense_out, vxg_report* report);

/* vxg_model_forward with the pooling realisation chosen per pool layer, as an
 * ExecutionPlan does (planner.hpp:94-125; PrimitiveKind pool_plain /
 * pool_fragments): pool_modes holds one entry per pool layer, 0 = max_pool
 * (plain), 1 = mpf_pool (fragments), NULL = the network's forced modes with
 * fragments where it leaves the choice.  A mode contradicting a forced one is
 * VXG_INVALID (planner.cpp:565-566).  dense_out has the plan's output shape:
 * fragment pools are recombined, plain pools subsample. */
int vxg_model_forward_ex(vxg_model* model, int mem, const float* input, int64_t S,
                         const int64_t e[3], const int* conv_algos, const int* pool_modes,
                         int cache_spectra, float* dense_out, vxg_report* report);

/* The device plan for (S, e) with explicit pool modes: per layer 8 int64
 * {kind (0 conv, 1 pool), conv algo or pool mode, tile T, tiles per entry,
 * tensor cores, measured, estimated ns, 0} into out (8 * layers; may be NULL),
 * and the peak HBM bytes of the forward into *bytes (may be NULL).  Works on a
 * planning-only model (vxg_model_create with weights == NULL). */
int vxg_model_plan_ex(vxg_model* model, int64_t S, const int64_t e[3], const int* conv_algos,
                      const int* pool_modes, int64_t* out, int64_t* bytes);

/* Streaming forward over `count` patches of the same shape (the tiler's
 * production path): double-buffered device tensors and two copy streams, so
 * the upload of patch k + 1 and the download of patch k - 1 overlap the
 * forward of patch k (pinned host buffers give true overlap).  seconds
 * (optional) = device time from the first upload to the last download. */
int vxg_model_forward_many(vxg_model* model, int64_t count, const float* const* inputs, int64_t S,
                           const int64_t e[3], const int* conv_algos, int cache_spectra,
                           float* const* outputs, double* seconds);

/* Measured-time planning: times the candidate tile sizes (and the direct
 * kernel where it may compete) for every conv layer of the plan of (S, e) on
 * sample inputs; later plans of this model choose per layer by measured cost. */
int vxg_model_tune(vxg_model* model, int64_t S, const int64_t e[3]);
/* The plan for (S, e) (conv_algos as vxg_model_forward): per layer 7 int64
 * {kind (0 conv, 1 pool), algo (vxg_conv_algo), tile size T, tiles per entry,
 * tensor cores, measured, estimated nanoseconds}; `out` holds 7 * layers. */
int vxg_model_plan_info(vxg_model* model, int64_t S, const int64_t e[3], const int* conv_algos,
                        int64_t* out);

/* Peak HBM bytes vxg_model_forward would need for input extent e (planner
 * feasibility), or -1 when the shape chain is invalid. */
int64_t vxg_model_plan_bytes(vxg_model* model, int64_t S, const int64_t e[3],
                             const int* conv_algos);

#ifdef __cplusplus
}
#endif

#endif /* VXG_H_ */
