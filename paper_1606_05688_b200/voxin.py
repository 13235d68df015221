"""Python mirror of the reference's layer-primitive and network-forward
interface (proj/include/voxin), backed by the sm_100a kernels of libvxg.so.

Names, argument meaning and error behaviour follow the reference:

==========================  =====================================================
this module                 reference
==========================  =====================================================
ConvLayerParams             layers.hpp:19-34
LayerResult / MemoryAudit   layers.hpp:37-40, memory.hpp:100-103
conv_direct                 layers.hpp:142-192
conv_fft_data_parallel      layers.hpp:203-272   (device: tiled pruned FFT)
conv_fft_staged             layers.hpp:286-371   (device: tiled pruned FFT)
conv_fft_task_parallel      task_conv.hpp:415-442 (device: tiled pruned FFT)
max_pool / mpf_pool         layers.hpp:377-470
recombine_fragments         layers.hpp:477-520
optimal_fft_size            fft.hpp:50-56
pruned_fft_forward/inverse  fft.hpp:391-414
batched_fft_forward/inverse fft.hpp:419-457
NetworkSpec / parse / fmt   network.hpp, netspec.cpp:54-151
field_of_view               cost.cpp:107-122
propagate_shapes            planner.cpp:536-589
random_weights              execute.hpp:50-73
fill_random                 cli.cpp:78-84
execute / Model.forward     execute.hpp:388-402 (all-fragment plan, device resident)
==========================  =====================================================

Tensors are float32 arrays in the Tensor5 layout (s, f, x, y, z).  A numpy
array runs through host staging (the call is synchronous); a CUDA
torch.Tensor is used in place (stream-ordered on the context's stream).
"""
from __future__ import annotations

import atexit
import ctypes as C
import threading
import weakref
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import ParseError, ResourceExhausted, check, i64s, lib

__all__ = [
    "Context", "default_context", "ConvLayerParams", "LayerResult", "MemoryAudit",
    "conv_direct", "conv_fft_data_parallel", "conv_fft_staged", "conv_fft_task_parallel",
    "conv", "max_pool", "mpf_pool", "recombine_fragments", "optimal_fft_size",
    "pruned_fft_forward", "pruned_fft_inverse", "batched_fft_forward", "batched_fft_inverse",
    "NetworkSpec", "parse_network_spec", "format_network_spec", "field_of_view",
    "propagate_shapes", "random_weights", "fill_random", "execute", "Model",
    "ThroughputReport", "ParseError", "ResourceExhausted",
    "conv_fft_tiled", "TILE_SIZES",
]


# ---- context ---------------------------------------------------------------------------


def _finish(ctx, mem):
    """Layer primitives are externally synchronous (the reference's contract,
    SPEC.md:283): device-pointer calls are stream-ordered inside the library,
    so wait for them before handing results back to the caller's streams."""
    if mem == L.MEM_DEVICE:
        ctx.sync()

_live_contexts = weakref.WeakSet()
_live_models = weakref.WeakSet()


@atexit.register
def _close_all_contexts():
    # before the CUDA runtime's own teardown at process exit; models first
    for m in list(_live_models):
        try:
            m.close()
        except Exception:
            pass
    for c in list(_live_contexts):
        try:
            c.close()
        except Exception:
            pass


class Context:
    """One per GPU: stream, stream-ordered allocator, HBM budget (bytes; <= 0: free HBM - 2.5 GiB)."""

    def __init__(self, device: int = 0, budget_bytes: int = 0):
        p = C.c_void_p()
        check(lib().vxg_ctx_create(int(device), int(budget_bytes), C.byref(p)))
        self._p = p
        self.device = device
        _live_contexts.add(self)

    @property
    def handle(self):
        return self._p

    def sync(self):
        check(lib().vxg_ctx_sync(self._p))

    def trim(self):
        """Give the forward's cached arena block and the pool's free memory back
        to the device (vxg_ctx_trim)."""
        check(lib().vxg_ctx_trim(self._p))

    def stream(self) -> int:
        s = C.c_void_p()
        check(lib().vxg_ctx_stream(self._p, C.byref(s)))
        return s.value or 0

    def memory(self):
        cur, peak, bud = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().vxg_ctx_memory(self._p, C.byref(cur), C.byref(peak), C.byref(bud)))
        return {"current": cur.value, "peak": peak.value, "budget": bud.value}

    def reset_peak(self):
        check(lib().vxg_ctx_reset_peak(self._p))

    @property
    def launches(self) -> int:
        return int(lib().vxg_ctx_launches(self._p))

    KERNEL_KINDS = ("tile_fwd", "tile_inv", "cgemm", "kspec", "direct", "pool", "recombine",
                    "linefft", "other")

    def profile(self, enable: bool):
        """Record CUDA events around every launch (per-kernel device time)."""
        check(lib().vxg_ctx_profile(self._p, 1 if enable else 0))

    def kernel_stats(self):
        """{kind: {launches, seconds, flops, bytes}} of the recorded launches."""
        out = {}
        for i, name in enumerate(self.KERNEL_KINDS):
            n = C.c_int64()
            s, fl, by = C.c_double(), C.c_double(), C.c_double()
            check(lib().vxg_ctx_kernel_stats(self._p, i, C.byref(n), C.byref(s), C.byref(fl),
                                             C.byref(by)))
            if n.value:
                out[name] = {"launches": n.value, "seconds": s.value, "flops": fl.value,
                             "bytes": by.value}
        return out

    def bench_ffma(self) -> float:
        t = C.c_double()
        check(lib().vxg_bench_ffma(self._p, C.byref(t)))
        return t.value

    def close(self):
        if self._p:
            lib().vxg_ctx_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: dict = {}
_default_lock = threading.Lock()


def default_context(device: int = 0) -> Context:
    with _default_lock:
        if device not in _default:
            _default[device] = Context(device)
        return _default[device]


# ---- tensors -----------------------------------------------------------------------------

def _is_torch_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


def _torch_ready(x):
    """The library runs on its own stream: torch work that produced (or last
    used the memory of) a CUDA tensor must be complete before it is handed over."""
    import torch
    torch.cuda.current_stream(x.device).synchronize()


class _Arg:
    """Resolves one tensor argument to (mem, pointer)."""

    def __init__(self, x, dtype=np.float32):
        if _is_torch_cuda(x):
            import torch
            if x.dtype != torch.float32 or not x.is_contiguous():
                raise ValueError("device tensors must be contiguous float32")
            _torch_ready(x)
            self.mem, self.ptr, self.keep = L.MEM_DEVICE, C.c_void_p(x.data_ptr()), x
        else:
            a = np.ascontiguousarray(x, dtype=dtype)
            self.mem, self.ptr, self.keep = L.MEM_HOST, a.ctypes.data_as(C.c_void_p), a


def _out_like(ref, shape, dtype=np.float32):
    if _is_torch_cuda(ref):
        import torch
        tdt = torch.float32 if dtype == np.float32 else torch.complex64
        return torch.empty(tuple(int(s) for s in shape), dtype=tdt, device=ref.device)
    return np.empty(tuple(int(s) for s in shape), dtype=dtype)


def _ptr_of(t):
    if _is_torch_cuda(t):
        _torch_ready(t)
        return C.c_void_p(t.data_ptr())
    return t.ctypes.data_as(C.c_void_p)


def _check_out(out, shape, like):
    """A caller-supplied output must match what the call writes: shape, float32,
    contiguous, and on the same side (host / device) as the input -- the C-ABI
    takes raw pointers and cannot check any of this itself."""
    shape = tuple(int(s) for s in shape)
    if _is_torch_cuda(like) != _is_torch_cuda(out):
        raise ValueError("out must live on the same side (host or device) as the input")
    if _is_torch_cuda(out):
        import torch
        if out.dtype != torch.float32 or not out.is_contiguous() or tuple(out.shape) != shape \
                or out.device != like.device:
            raise ValueError(f"out must be a contiguous float32 CUDA tensor of shape {shape} "
                             "on the input's device")
    else:
        if not isinstance(out, np.ndarray) or out.dtype != np.float32 or not out.flags.c_contiguous \
                or tuple(out.shape) != shape or not out.flags.writeable:
            raise ValueError(f"out must be a writeable C-contiguous float32 array of shape {shape}")
    return out


def _check_weights(net, weights):
    """NetworkWeights check (execute.hpp: one kernel set + bias per conv layer):
    the flat weight vector must hold exactly net.weight_count() scalars."""
    n = int(np.prod(weights.shape)) if hasattr(weights, "shape") else len(weights)
    if n != net.weight_count():
        raise ValueError(f"weights: {n} scalars given, the network needs {net.weight_count()}")


def _same_mem(*args):
    mems = {a.mem for a in args}
    if len(mems) != 1:
        raise ValueError("all tensors of one call must live on the same side (host or device)")
    return mems.pop()


# ---- layer primitives ------------------------------------------------------------------------

@dataclass
class MemoryAudit:
    peak: float = 0.0
    model: float = 0.0


@dataclass
class LayerResult:
    output: object
    audit: MemoryAudit = field(default_factory=MemoryAudit)


@dataclass
class ConvLayerParams:
    """kernels (f_out, f_in, kx, ky, kz), bias (f_out,), act 'relu' | 'identity'."""
    kernels: object
    bias: object
    act: str = "identity"

    def features_out(self) -> int:
        return int(self.kernels.shape[0])

    def features_in(self) -> int:
        return int(self.kernels.shape[1])

    def kernel_extents(self):
        return tuple(int(v) for v in self.kernels.shape[2:])


def conv(input, params: ConvLayerParams, algo: int = L.CONV_AUTO, ctx: Optional[Context] = None):
    ctx = ctx or default_context()
    if len(input.shape) != 5 or len(params.kernels.shape) != 5:
        raise ValueError("conv: input and kernels must be 5D (s, f, x, y, z)")
    S, f = int(input.shape[0]), int(input.shape[1])
    n = [int(v) for v in input.shape[2:]]
    fo = params.features_out()
    k = params.kernel_extents()
    if params.features_in() != f:
        raise ValueError("conv: kernel feature count mismatch")
    if int(np.prod(params.bias.shape)) != fo:
        raise ValueError("conv: bias count mismatch")
    if any(k[a] > n[a] for a in range(3)):
        raise ValueError("conv: kernel larger than image")
    xi, wi, bi = _Arg(input), _Arg(params.kernels), _Arg(params.bias)
    mem = _same_mem(xi, wi, bi)
    out = _out_like(input, (S, fo) + tuple(n[a] - k[a] + 1 for a in range(3)))
    au = L.Audit()
    check(lib().vxg_conv(ctx.handle, int(algo), mem, xi.ptr, S, f, i64s(n), wi.ptr, fo, i64s(k),
                         bi.ptr, 1 if params.act == "relu" else 0, _ptr_of(out), C.byref(au)))
    _finish(ctx, mem)
    return LayerResult(out, MemoryAudit(au.peak, au.model))


def conv_direct(input, params, ctx=None, variant="naive"):
    """conv_direct (layers.hpp:142-192); both DirectVariant values use one device kernel."""
    return conv(input, params, L.CONV_DIRECT, ctx)


def conv_fft_data_parallel(input, params, ctx=None):
    return conv(input, params, L.CONV_FFT, ctx)


def conv_fft_staged(input, params, ctx=None):
    return conv(input, params, L.CONV_FFT, ctx)


def conv_fft_task_parallel(input, params, ctx=None):
    return conv(input, params, L.CONV_FFT, ctx)


def conv_fft_tiled(input, params: ConvLayerParams, tile: int, tensor_cores: bool = True,
                   cta_pair: bool = True, spectra_budget: int = 0, ctx: Optional[Context] = None):
    """The tiled FFT convolution with its plan pinned (vxg_conv_fft_tiled): tile FFT
    size, tcgen05 vs FFMA contraction, CTA-pair vs one-CTA forward transform."""
    ctx = ctx or default_context()
    S, f = int(input.shape[0]), int(input.shape[1])
    n = [int(v) for v in input.shape[2:]]
    fo = params.features_out()
    k = params.kernel_extents()
    xi, wi, bi = _Arg(input), _Arg(params.kernels), _Arg(params.bias)
    mem = _same_mem(xi, wi, bi)
    out = _out_like(input, (S, fo) + tuple(n[a] - k[a] + 1 for a in range(3)))
    flags = (0 if tensor_cores else 1) | (0 if cta_pair else 2)
    check(lib().vxg_conv_fft_tiled(ctx.handle, mem, xi.ptr, S, f, i64s(n), wi.ptr, fo, i64s(k), bi.ptr,
                                   1 if params.act == "relu" else 0, _ptr_of(out), int(tile), flags,
                                   int(spectra_budget)))
    _finish(ctx, mem)
    return out


TILE_SIZES = (4, 6, 8, 10, 12, 16, 20, 24, 28, 30, 32, 36, 40)  # 36, 40: CTA pairs (k_tilefft.cu)


def _pool(fn, input, p, P, ctx):
    ctx = ctx or default_context()
    if len(input.shape) != 5:
        raise ValueError("pool: input must be 5D")
    p = [int(v) for v in (p if isinstance(p, (list, tuple)) else (p, p, p))]
    if any(v <= 0 for v in p):
        raise ValueError("pool: window extents must be positive")
    S, f = int(input.shape[0]), int(input.shape[1])
    n = [int(v) for v in input.shape[2:]]
    xi = _Arg(input)
    out = _out_like(input, (S * (int(np.prod(p)) if P else 1), f) + tuple(n[a] // p[a] for a in range(3)))
    au = L.Audit()
    check(fn(ctx.handle, xi.mem, xi.ptr, S, f, i64s(n), i64s(p), _ptr_of(out), C.byref(au)))
    _finish(ctx, xi.mem)
    return LayerResult(out, MemoryAudit(au.peak, au.model))


def max_pool(input, p, ctx=None):
    return _pool(lib().vxg_max_pool, input, p, False, ctx)


def mpf_pool(input, p, ctx=None):
    return _pool(lib().vxg_mpf_pool, input, p, True, ctx)


def recombine_fragments(fragments, windows: Sequence[Sequence[int]], original_batch: int,
                        ctx=None):
    ctx = ctx or default_context()
    S, f = int(fragments.shape[0]), int(fragments.shape[1])
    n = [int(v) for v in fragments.shape[2:]]
    stride = [1, 1, 1]
    flat = []
    for w in windows:
        w = [int(v) for v in w]
        if any(v <= 0 for v in w):
            raise ValueError("recombine_fragments: bad window")
        stride = [stride[a] * w[a] for a in range(3)]
        flat += w
    xi = _Arg(fragments)
    out = _out_like(fragments, (int(original_batch), f) + tuple(stride[a] * n[a] for a in range(3)))
    check(lib().vxg_recombine(ctx.handle, xi.mem, xi.ptr, S, f, i64s(n), i64s(flat), len(windows),
                              int(original_batch), _ptr_of(out)))
    _finish(ctx, xi.mem)
    return out


# ---- transforms --------------------------------------------------------------------------------

_PROFILES = {"host": L.PROFILE_HOST, "device": L.PROFILE_DEVICE, "any": L.PROFILE_ANY}


def optimal_fft_size(n: int, profile: str = "host") -> int:
    if n <= 0:
        raise ValueError("optimal_fft_size: n must be positive")
    return int(lib().vxg_optimal_fft_size(int(n), _PROFILES[profile]))


def _complex_out(ref, shape):
    if _is_torch_cuda(ref):
        import torch
        return torch.empty(tuple(shape), dtype=torch.complex64, device=ref.device)
    return np.empty(tuple(shape), dtype=np.complex64)


def pruned_fft_forward(img, padded, ctx=None):
    """Single-image transform; result (floor(px/2)+1, py, pz) complex64."""
    ctx = ctx or default_context()
    n = [int(v) for v in img.shape[-3:]]
    p = [int(v) for v in padded]
    xi = _Arg(img)
    out = _complex_out(img, (p[0] // 2 + 1, p[1], p[2]))
    check(lib().vxg_fft_pruned_forward(ctx.handle, xi.mem, xi.ptr, i64s(n), i64s(p), _ptr_of(out)))
    _finish(ctx, xi.mem)
    return out


def pruned_fft_inverse(spec, padded, crop, ctx=None):
    ctx = ctx or default_context()
    p = [int(v) for v in padded]
    c = [int(v) for v in crop]
    xi = _Arg(spec, np.complex64)
    out = _out_like(spec, tuple(c))
    check(lib().vxg_fft_pruned_inverse(ctx.handle, xi.mem, xi.ptr, i64s(p), i64s(c), _ptr_of(out)))
    _finish(ctx, xi.mem)
    return out


def batched_fft_forward(imgs, padded, ctx=None):
    """b images (b, x, y, z) -> (b, floor(pz/2)+1, py, px) complex64 (permuted layout)."""
    ctx = ctx or default_context()
    b = int(imgs.shape[0])
    n = [int(v) for v in imgs.shape[-3:]]
    p = [int(v) for v in padded]
    xi = _Arg(imgs)
    out = _complex_out(imgs, (b, p[2] // 2 + 1, p[1], p[0]))
    check(lib().vxg_fft_batched_forward(ctx.handle, xi.mem, xi.ptr, b, i64s(n), i64s(p), _ptr_of(out)))
    _finish(ctx, xi.mem)
    return out


def batched_fft_inverse(spec, padded, crop, ctx=None):
    ctx = ctx or default_context()
    b = int(spec.shape[0])
    p = [int(v) for v in padded]
    c = [int(v) for v in crop]
    xi = _Arg(spec, np.complex64)
    out = _out_like(spec, (b,) + tuple(c))
    check(lib().vxg_fft_batched_inverse(ctx.handle, xi.mem, xi.ptr, b, i64s(p), i64s(c), _ptr_of(out)))
    _finish(ctx, xi.mem)
    return out


# ---- networks ------------------------------------------------------------------------------------

class NetworkSpec:
    """Parsed network description (network.hpp:32-65)."""

    def __init__(self, text: str):
        p = C.c_void_p()
        check(lib().vxg_net_parse(text.encode(), C.byref(p)))
        self._p = p
        info = (C.c_int64 * 5)()
        check(lib().vxg_net_info(self._p, info))
        self.layer_count, self.conv_count, self.pool_count, self.features_in, self.features_out = list(info)
        self.layers = []
        for l in range(self.layer_count):
            kind, fo, relu, forced = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
            ext = (C.c_int64 * 3)()
            check(lib().vxg_net_layer(self._p, l, C.byref(kind), ext, C.byref(fo), C.byref(relu),
                                      C.byref(forced)))
            if kind.value == 0:
                self.layers.append(("conv", fo.value, tuple(ext), bool(relu.value)))
            else:
                mode = {-1: "auto", 0: "plain", 1: "mpf"}[forced.value]
                self.layers.append(("pool", tuple(ext), mode))

    @property
    def handle(self):
        return self._p

    def format(self) -> str:
        need = C.c_int64()
        check(lib().vxg_net_format(self._p, None, 0, C.byref(need)))
        buf = C.create_string_buffer(int(need.value))
        check(lib().vxg_net_format(self._p, buf, need.value, C.byref(need)))
        return buf.value.decode()

    def field_of_view(self):
        v = (C.c_int64 * 3)()
        check(lib().vxg_net_fov(self._p, v))
        return tuple(v)

    def weight_count(self) -> int:
        return int(lib().vxg_net_weight_count(self._p))

    def propagate(self, S: int, e, modes=None):
        """(shapes list of (s,f,x,y,z), violation layer or -1)."""
        e = [int(v) for v in (e if isinstance(e, (list, tuple)) else (e, e, e))]
        shapes = (C.c_int64 * (5 * (self.layer_count + 1)))()
        viol = C.c_int64()
        m = None
        if modes is not None:
            m = (C.c_int * max(1, len(modes)))(*[int(x) for x in modes])
        check(lib().vxg_net_propagate(self._p, int(S), i64s(e), m, shapes, C.byref(viol)))
        n = self.layer_count + 1 if viol.value < 0 else viol.value + 1
        return [tuple(shapes[5 * i:5 * i + 5]) for i in range(n)], viol.value

    def __del__(self):
        try:
            if self._p:
                lib().vxg_net_free(self._p)
                self._p = None
        except Exception:
            pass


def parse_network_spec(text: str) -> NetworkSpec:
    return NetworkSpec(text)


def format_network_spec(net: NetworkSpec) -> str:
    return net.format()


def field_of_view(net: NetworkSpec):
    return net.field_of_view()


def propagate_shapes(net: NetworkSpec, input_shape, pool_modes=None):
    s, f, x, y, z = input_shape
    if f != net.features_in:
        raise ValueError("propagate_shapes: input features must match the network")
    return net.propagate(s, (x, y, z), pool_modes)


def random_weights(net: NetworkSpec, seed: int) -> np.ndarray:
    """Flat float32: per conv layer kernels (fo, f, k) then biases (fo)."""
    w = np.empty(net.weight_count(), np.float32)
    check(lib().vxg_random_weights(net.handle, C.c_uint64(seed), w.ctypes.data_as(C.c_void_p)))
    return w


def conv_params(net: NetworkSpec, flat: np.ndarray):
    """Split flat weights into ConvLayerParams per conv layer."""
    out, off, f = [], 0, net.features_in
    for l in net.layers:
        if l[0] != "conv":
            continue
        fo, k, relu = l[1], l[2], l[3]
        nk = fo * f * int(np.prod(k))
        ker = flat[off:off + nk].reshape((fo, f) + tuple(k))
        off += nk
        b = flat[off:off + fo]
        off += fo
        out.append(ConvLayerParams(ker, b, "relu" if relu else "identity"))
        f = fo
    return out


def fill_random(count_or_shape, seed: int) -> np.ndarray:
    shape = (count_or_shape,) if isinstance(count_or_shape, int) else tuple(count_or_shape)
    a = np.empty(int(np.prod(shape)), np.float32)
    check(lib().vxg_fill_random(a.ctypes.data_as(C.c_void_p), a.size, C.c_uint64(seed)))
    return a.reshape(shape)


@dataclass
class ThroughputReport:
    """execute.hpp:76-84 (device flavour: CUDA-event seconds)."""
    voxels: float
    seconds: float
    voxels_per_second: float
    device_peak: float
    layer_seconds: list


def _report(r: L.Report) -> ThroughputReport:
    return ThroughputReport(r.voxels, r.seconds, r.voxels_per_second, r.device_peak,
                            [r.layer_seconds[i] for i in range(r.layers)])


def _algos(net: NetworkSpec, conv_algos):
    if conv_algos is None:
        return None
    if isinstance(conv_algos, (str, int)):
        conv_algos = [conv_algos] * net.conv_count
    names = {"auto": L.CONV_AUTO, "direct": L.CONV_DIRECT, "fft": L.CONV_FFT}
    vals = [names[a] if isinstance(a, str) else int(a) for a in conv_algos]
    if len(vals) != net.conv_count:
        raise ValueError("one algorithm per conv layer required")
    return (C.c_int * len(vals))(*vals)


class Model:
    """Device-resident weights of one network (kernel spectra cached per tile size)."""

    def __init__(self, net: NetworkSpec, weights, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.net = net
        _check_weights(net, weights)
        wi = _Arg(weights)
        p = C.c_void_p()
        check(lib().vxg_model_create(self.ctx.handle, net.handle, wi.ptr, wi.mem, C.byref(p)))
        self._p = p
        _live_models.add(self)

    def output_shape(self, S: int, e):
        e = [int(v) for v in (e if isinstance(e, (list, tuple)) else (e, e, e))]
        fov = self.net.field_of_view()
        return (int(S), self.net.features_out) + tuple(e[a] - fov[a] + 1 for a in range(3))

    def plan_bytes(self, S: int, e, conv_algos=None) -> int:
        e = [int(v) for v in (e if isinstance(e, (list, tuple)) else (e, e, e))]
        return int(lib().vxg_model_plan_bytes(self._p, int(S), i64s(e), _algos(self.net, conv_algos)))

    def forward_many(self, inputs, outputs=None, conv_algos=None, cache_spectra=True):
        """Streaming forward over host patches of one shape (vxg_model_forward_many):
        uploads / downloads overlap the forwards.  inputs: list of (S, f_in, *e)
        float32 host arrays (pinned for true overlap); returns (outputs, seconds)."""
        if not inputs:
            return [], 0.0
        S = int(inputs[0].shape[0])
        e = [int(v) for v in inputs[0].shape[2:]]
        shape = self.output_shape(S, e)
        if outputs is None:
            outputs = [np.empty(shape, np.float32) for _ in inputs]
        for x in inputs:
            if tuple(x.shape) != tuple(inputs[0].shape) or x.dtype != np.float32 or not x.flags.c_contiguous:
                raise ValueError("forward_many: inputs must be C-contiguous float32 of one shape")
        for y in outputs:
            if tuple(y.shape) != shape or y.dtype != np.float32 or not y.flags.c_contiguous:
                raise ValueError("forward_many: outputs must be C-contiguous float32 of the output shape")
        ins = (C.c_void_p * len(inputs))(*[x.ctypes.data for x in inputs])
        outs = (C.c_void_p * len(outputs))(*[y.ctypes.data for y in outputs])
        sec = C.c_double()
        check(lib().vxg_model_forward_many(self._p, len(inputs), ins, S, i64s(e),
                                           _algos(self.net, conv_algos), 1 if cache_spectra else 0, outs,
                                           C.byref(sec)))
        return outputs, sec.value

    def tune(self, S: int, e):
        """Measured-time planning for input (S, f_in, e) (vxg_model_tune)."""
        e = [int(v) for v in (e if isinstance(e, (list, tuple)) else (e, e, e))]
        check(lib().vxg_model_tune(self._p, int(S), i64s(e)))

    def plan_info(self, S: int, e, conv_algos=None):
        """Per layer: {"kind", "algo", "T", "tiles", "tc", "measured", "seconds"} of the
        plan for (S, e); "seconds" is the planner's estimate (measured costs after tune())."""
        e = [int(v) for v in (e if isinstance(e, (list, tuple)) else (e, e, e))]
        n = self.net.layer_count
        buf = (C.c_int64 * (7 * n))()
        check(lib().vxg_model_plan_info(self._p, int(S), i64s(e), _algos(self.net, conv_algos), buf))
        algo = {L.CONV_DIRECT: "direct", L.CONV_FFT: "fft"}
        out = []
        for i in range(n):
            k, a, T, tiles, tc, meas, ns = buf[7 * i:7 * i + 7]
            if k == 0:
                out.append({"layer": i, "kind": "conv", "algo": algo.get(a, str(a)), "T": T,
                            "tiles": tiles, "tc": bool(tc), "tc_tiles": {1: "quad", 2: "pair"}.get(int(tc)),
                            "measured": bool(meas), "seconds": ns * 1e-9})
            else:
                out.append({"layer": i, "kind": "pool", "seconds": ns * 1e-9})
        return out

    def forward(self, input, out=None, conv_algos=None, cache_spectra=True):
        S = int(input.shape[0])
        e = [int(v) for v in input.shape[2:]]
        if int(input.shape[1]) != self.net.features_in:
            raise ValueError("execute: input does not match the network")
        if len(input.shape) != 5:
            raise ValueError("execute: input must be 5D (s, f, x, y, z)")
        xi = _Arg(input)
        if out is None:
            out = _out_like(input, self.output_shape(S, e))
        else:
            _check_out(out, self.output_shape(S, e), input)
        rep = L.Report()
        check(lib().vxg_model_forward(self._p, xi.mem, xi.ptr, S, i64s(e), _algos(self.net, conv_algos),
                                      1 if cache_spectra else 0, _ptr_of(out), C.byref(rep)))
        return out, _report(rep)

    def close(self):
        if getattr(self, "_p", None):
            lib().vxg_model_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def execute(net: NetworkSpec, weights, input, ctx: Optional[Context] = None, conv_algos=None):
    """execute_plan (execute.hpp:388-402) with an all-fragment plan: (dense, report)."""
    ctx = ctx or default_context()
    if len(input.shape) != 5 or int(input.shape[1]) != net.features_in:
        raise ValueError("execute: input does not match the network")
    _check_weights(net, weights)
    S = int(input.shape[0])
    e = [int(v) for v in input.shape[2:]]
    wi, xi = _Arg(weights), _Arg(input)
    mem = _same_mem(wi, xi)
    fov = net.field_of_view()
    out = _out_like(input, (S, net.features_out) + tuple(e[a] - fov[a] + 1 for a in range(3)))
    rep = L.Report()
    check(lib().vxg_net_forward(ctx.handle, net.handle, wi.ptr, mem, xi.ptr, S, i64s(e),
                                _algos(net, conv_algos), _ptr_of(out), C.byref(rep)))
    return out, _report(rep)
