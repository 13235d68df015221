"""ctypes binding of libvxg.so (the C-ABI in include/vxg.h).

The shared library is built in-tree by ``python -m paper_1606_05688_b200.build``
(or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libvxg.so"

OK, INVALID, EXHAUSTED, CUDA, PARSE, INTERNAL = 0, 1, 2, 3, 4, 5
MEM_HOST, MEM_DEVICE = 0, 1
CONV_AUTO, CONV_DIRECT, CONV_FFT = 0, 1, 2
PROFILE_HOST, PROFILE_DEVICE, PROFILE_ANY = 0, 1, 2


class ResourceExhausted(MemoryError):
    """vx::resource_exhausted (proj/include/voxin/common.hpp:12-14)."""


class ParseError(RuntimeError):
    """vx::ParseError (proj/include/voxin/netspec.hpp:11-20): carries the line."""

    def __init__(self, msg: str):
        super().__init__(msg)
        self.line = None
        if msg.startswith("line "):
            try:
                self.line = int(msg.split(":")[0].split()[1])
            except (IndexError, ValueError):
                pass


class CudaError(RuntimeError):
    pass


class Audit(C.Structure):
    _fields_ = [("peak", C.c_double), ("model", C.c_double)]


class Report(C.Structure):
    _fields_ = [("voxels", C.c_double), ("seconds", C.c_double),
                ("voxels_per_second", C.c_double), ("device_peak", C.c_double),
                ("layers", C.c_int64), ("layer_seconds", C.c_double * 64)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is not built: run `python -m paper_1606_05688_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    P = C.c_void_p
    I64 = C.c_int64
    I = C.c_int
    A = C.POINTER(C.c_int64)
    sigs = {
        "vxg_last_error": (C.c_char_p, []),
        "vxg_version": (C.c_char_p, []),
        "vxg_ctx_create": (I, [I, I64, C.POINTER(P)]),
        "vxg_ctx_destroy": (I, [P]),
        "vxg_ctx_sync": (I, [P]),
        "vxg_ctx_trim": (I, [P]),
        "vxg_ctx_stream": (I, [P, C.POINTER(P)]),
        "vxg_ctx_memory": (I, [P, A, A, A]),
        "vxg_ctx_reset_peak": (I, [P]),
        "vxg_ctx_launches": (I64, [P]),
        "vxg_ctx_profile": (I, [P, I]),
        "vxg_ctx_kernel_stats": (I, [P, I, A, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]),
        "vxg_bench_ffma": (I, [P, C.POINTER(C.c_double)]),
        "vxg_conv": (I, [P, I, I, P, I64, I64, A, P, I64, A, P, I, P, C.POINTER(Audit)]),
        "vxg_conv_fft_tiled": (I, [P, I, P, I64, I64, A, P, I64, A, P, I, P, I, I, I64]),
        "vxg_max_pool": (I, [P, I, P, I64, I64, A, A, P, C.POINTER(Audit)]),
        "vxg_mpf_pool": (I, [P, I, P, I64, I64, A, A, P, C.POINTER(Audit)]),
        "vxg_recombine": (I, [P, I, P, I64, I64, A, A, I64, I64, P]),
        "vxg_optimal_fft_size": (I64, [I64, I]),
        "vxg_fft_pruned_forward": (I, [P, I, P, A, A, P]),
        "vxg_fft_pruned_inverse": (I, [P, I, P, A, A, P]),
        "vxg_fft_batched_forward": (I, [P, I, P, I64, A, A, P]),
        "vxg_fft_batched_inverse": (I, [P, I, P, I64, A, A, P]),
        "vxg_net_parse": (I, [C.c_char_p, C.POINTER(P)]),
        "vxg_net_free": (I, [P]),
        "vxg_net_format": (I, [P, C.c_char_p, I64, A]),
        "vxg_net_info": (I, [P, A]),
        "vxg_net_layer": (I, [P, I64, A, A, A, A, A]),
        "vxg_net_fov": (I, [P, A]),
        "vxg_net_propagate": (I, [P, I64, A, C.POINTER(I), A, A]),
        "vxg_net_weight_count": (I64, [P]),
        "vxg_random_weights": (I, [P, C.c_uint64, P]),
        "vxg_fill_random": (I, [P, I64, C.c_uint64]),
        "vxg_net_forward": (I, [P, P, P, I, P, I64, A, C.POINTER(I), P, C.POINTER(Report)]),
        "vxg_model_create": (I, [P, P, P, I, C.POINTER(P)]),
        "vxg_model_tune": (I, [P, I64, A]),
        "vxg_model_forward_many": (I, [P, I64, C.POINTER(P), I64, A, C.POINTER(I), I, C.POINTER(P),
                                       C.POINTER(C.c_double)]),
        "vxg_model_plan_info": (I, [P, I64, A, C.POINTER(I), A]),
        "vxg_model_free": (I, [P]),
        "vxg_model_forward": (I, [P, I, P, I64, A, C.POINTER(I), I, P, C.POINTER(Report)]),
        "vxg_model_plan_bytes": (I64, [P, I64, A, C.POINTER(I)]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().vxg_last_error().decode()
    if rc == INVALID:
        raise ValueError(msg)
    if rc == EXHAUSTED:
        raise ResourceExhausted(msg)
    if rc == PARSE:
        raise ParseError(msg)
    if rc == CUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)


def i64s(v) -> "C.Array":
    v = [int(x) for x in v]
    return (C.c_int64 * max(1, len(v)))(*v)
