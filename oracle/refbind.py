"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the two checkers.

* ``Ref``    — oracle/_ref/libvoxref.so, the UNMODIFIED reference library
               (built from /root/reference/proj by oracle/build_ref.sh).
* ``Oracle`` — oracle/_build/liboracle.so, the plain-C restatement
               (oracle/voxin_oracle.c), pinned against the reference by
               tests/test_oracle.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libvoxref.so"
ORACLE_SO = HERE / "_build" / "liboracle.so"

_i64p = C.POINTER(C.c_int64)


def _a64(v):
    return (C.c_int64 * len(v))(*[int(x) for x in v])


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def build_oracle() -> Path:
    """Compile the C restatement (cheap; also done by __graft_entry__.build())."""
    src = HERE / "voxin_oracle.c"
    ORACLE_SO.parent.mkdir(parents=True, exist_ok=True)
    if not ORACLE_SO.exists() or ORACLE_SO.stat().st_mtime < src.stat().st_mtime:
        tmp = ORACLE_SO.with_suffix(".so.tmp")
        rc = os.system(f"gcc -O3 -fPIC -shared -o {tmp} {src} -lm")
        if rc != 0:
            raise RuntimeError("failed to compile oracle/voxin_oracle.c")
        os.replace(tmp, ORACLE_SO)
    return ORACLE_SO


class Ref:
    """The reference implementation itself (fp32 or fp64)."""

    def __init__(self, workers: int = 0):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} missing: run oracle/build_ref.sh")
        self.lib = C.CDLL(str(REF_SO))
        self.lib.ref_last_error.restype = C.c_char_p
        self.lib.ref_optimal_fft_size.restype = C.c_int64
        L, I, P, V, U, D = C.c_int64, C.c_int, _i64p, C.c_void_p, C.c_uint64, C.POINTER(C.c_double)
        sig = {
            "ref_conv": [I, I, V, L, L, P, V, L, P, V, I, V],
            "ref_pool": [I, I, V, L, L, P, P, V],
            "ref_recombine": [I, V, L, L, P, P, L, L, V],
            "ref_pruned_fwd": [I, V, P, P, V],
            "ref_pruned_inv": [I, V, P, P, V],
            "ref_batched_fwd": [I, V, L, P, P, V],
            "ref_batched_inv": [I, V, L, P, P, V],
            "ref_optimal_fft_size": [L, I],
            "ref_fov": [C.c_char_p, P],
            "ref_propagate": [C.c_char_p, L, P, C.POINTER(C.c_int), P, P],
            "ref_random_weights": [C.c_char_p, U, I, V],
            "ref_fill_random": [I, V, L, U],
            "ref_net_forward": [C.c_char_p, I, U, V, L, P, I, I, V, D],
            "ref_net_sample": [C.c_char_p, L, U, U, I, L, D, D, D],
            "ref_stepper_create": [C.c_char_p, L, U, U, I, I, C.POINTER(C.c_void_p), C.POINTER(C.c_int)],
            "ref_stepper_step": [V, P, D, C.POINTER(C.c_int)],
            "ref_stepper_output": [V, V, P],
            "ref_stepper_free": [V],
        }
        for name, args in sig.items():
            getattr(self.lib, name).argtypes = args
        self.workers = self.lib.ref_set_workers(int(workers))

    def _check(self, rc):
        if rc != 0:
            msg = self.lib.ref_last_error().decode()
            if rc == 1:
                raise ValueError(msg)
            if rc == 2:
                raise MemoryError(msg)
            raise RuntimeError(msg)

    @staticmethod
    def _dt(prec):
        return np.float64 if prec == 64 else np.float32

    def conv(self, kind, x, w, bias, relu, prec=64):
        dt = self._dt(prec)
        x = np.ascontiguousarray(x, dt)
        w = np.ascontiguousarray(w, dt)
        bias = np.ascontiguousarray(bias, dt)
        S, f = x.shape[:2]
        n = x.shape[2:]
        fo = w.shape[0]
        k = w.shape[2:]
        out = np.zeros((S, fo) + tuple(n[a] - k[a] + 1 for a in range(3)), dt)
        self._check(self.lib.ref_conv(int(kind), prec, _ptr(x), S, f, _a64(n), _ptr(w), fo,
                                      _a64(k), _ptr(bias), int(relu), _ptr(out)))
        return out

    def pool(self, fragments, x, p, prec=64):
        dt = self._dt(prec)
        x = np.ascontiguousarray(x, dt)
        S, f = x.shape[:2]
        n = x.shape[2:]
        no = tuple(n[a] // p[a] for a in range(3))
        P = int(np.prod(p)) if fragments else 1
        out = np.zeros((S * P, f) + no, dt)
        self._check(self.lib.ref_pool(int(fragments), prec, _ptr(x), S, f, _a64(n), _a64(p),
                                      _ptr(out)))
        return out

    def recombine(self, frag, windows, original_batch, prec=64):
        dt = self._dt(prec)
        frag = np.ascontiguousarray(frag, dt)
        S, f = frag.shape[:2]
        n = frag.shape[2:]
        stride = [1, 1, 1]
        for w in windows:
            stride = [stride[a] * w[a] for a in range(3)]
        out = np.zeros((original_batch, f) + tuple(stride[a] * n[a] for a in range(3)), dt)
        flat = [v for w in windows for v in w]
        self._check(self.lib.ref_recombine(prec, _ptr(frag), S, f, _a64(n), _a64(flat or [0]),
                                           len(windows), original_batch, _ptr(out)))
        return out

    def pruned_fwd(self, img, pad, prec=64):
        dt = self._dt(prec)
        img = np.ascontiguousarray(img, dt)
        ct = np.complex128 if prec == 64 else np.complex64
        out = np.zeros((pad[0] // 2 + 1, pad[1], pad[2]), ct)
        self._check(self.lib.ref_pruned_fwd(prec, _ptr(img), _a64(img.shape), _a64(pad), _ptr(out)))
        return out

    def pruned_inv(self, spec, pad, crop, prec=64):
        dt = self._dt(prec)
        ct = np.complex128 if prec == 64 else np.complex64
        spec = np.ascontiguousarray(spec, ct)
        out = np.zeros(tuple(crop), dt)
        self._check(self.lib.ref_pruned_inv(prec, _ptr(spec), _a64(pad), _a64(crop), _ptr(out)))
        return out

    def batched_fwd(self, imgs, pad, prec=64):
        dt = self._dt(prec)
        imgs = np.ascontiguousarray(imgs, dt)
        b = imgs.shape[0]
        ct = np.complex128 if prec == 64 else np.complex64
        out = np.zeros((b, pad[2] // 2 + 1, pad[1], pad[0]), ct)
        self._check(self.lib.ref_batched_fwd(prec, _ptr(imgs), b, _a64(imgs.shape[1:]), _a64(pad),
                                             _ptr(out)))
        return out

    def batched_inv(self, spec, pad, crop, prec=64):
        dt = self._dt(prec)
        ct = np.complex128 if prec == 64 else np.complex64
        spec = np.ascontiguousarray(spec, ct)
        b = spec.shape[0]
        out = np.zeros((b,) + tuple(crop), dt)
        self._check(self.lib.ref_batched_inv(prec, _ptr(spec), b, _a64(pad), _a64(crop), _ptr(out)))
        return out

    def optimal_fft_size(self, n, profile):
        return int(self.lib.ref_optimal_fft_size(int(n), int(profile)))

    def fov(self, net_text):
        out = (C.c_int64 * 3)()
        self._check(self.lib.ref_fov(net_text.encode(), out))
        return tuple(out)

    def propagate(self, net_text, nlayers, npools, S, e, modes):
        shapes = np.zeros((nlayers + 1, 5), np.int64)
        viol = C.c_int64(0)
        m = (C.c_int * max(1, npools))(*modes)
        self._check(self.lib.ref_propagate(net_text.encode(), S, _a64(e), m,
                                           shapes.ctypes.data_as(_i64p), C.byref(viol)))
        return shapes, viol.value

    def random_weights(self, net_text, seed, count, prec=32):
        out = np.zeros(count, self._dt(prec))
        self._check(self.lib.ref_random_weights(net_text.encode(), seed, prec, _ptr(out)))
        return out

    def fill_random(self, count, seed, prec=32):
        out = np.zeros(count, self._dt(prec))
        self._check(self.lib.ref_fill_random(prec, _ptr(out), count, seed))
        return out

    def net_forward(self, net_text, wseed, x, conv_kind=3, mpf=True, prec=64, out_shape=None):
        dt = self._dt(prec)
        x = np.ascontiguousarray(x, dt)
        out = np.zeros(out_shape, dt)
        secs = C.c_double(0)
        self._check(self.lib.ref_net_forward(net_text.encode(), prec, C.c_uint64(wseed), _ptr(x),
                                             x.shape[0], _a64(x.shape[2:]), int(conv_kind),
                                             int(mpf), _ptr(out), C.byref(secs)))
        return out, secs.value

    def net_sample(self, net_text, e, wseed, iseed, conv_kind=3, keep=1):
        ext, spent, vox = C.c_double(), C.c_double(), C.c_double()
        self._check(self.lib.ref_net_sample(net_text.encode(), int(e), C.c_uint64(wseed),
                                            C.c_uint64(iseed), int(conv_kind), int(keep),
                                            C.byref(ext), C.byref(spent), C.byref(vox)))
        return ext.value, spent.value, vox.value


    # PrimitiveKind (proj/include/voxin/cost.hpp:13-24)
    KINDS = ("direct-naive", "direct-temp", "fft-data-parallel", "fft-task-parallel", "fft-staged",
             "device-direct-default", "device-direct-precomp", "device-fft", "pool-plain", "pool-fragments")

    def stepper(self, net_text, e, wseed, iseed, plan="forced", conv_kind=3, nlayers=64):
        """execute_plan's host-only path one layer per step (ref_stepper_*):
        plan="planner" -> the reference's own optimize_plan at extent e,
        plan="forced"  -> every conv = conv_kind, every pool MPF."""
        return RefStepper(self, net_text, e, wseed, iseed, plan, conv_kind, nlayers)


class RefStepper:
    def __init__(self, ref, net_text, e, wseed, iseed, plan, conv_kind, nlayers):
        self.ref = ref
        self.h = C.c_void_p()
        kinds = (C.c_int * nlayers)(*([-1] * nlayers))
        ref._check(ref.lib.ref_stepper_create(net_text.encode(), int(e), C.c_uint64(wseed), C.c_uint64(iseed),
                                              0 if plan == "planner" else 1, int(conv_kind), C.byref(self.h), kinds))
        self.kinds = [Ref.KINDS[k] for k in kinds if k >= 0]

    def step(self):
        """-> (layer, seconds, done)"""
        li, sec, done = C.c_int64(), C.c_double(), C.c_int()
        self.ref._check(self.ref.lib.ref_stepper_step(self.h, C.byref(li), C.byref(sec), C.byref(done)))
        return li.value, sec.value, bool(done.value)

    def output(self):
        sh = (C.c_int64 * 5)()
        self.ref._check(self.ref.lib.ref_stepper_output(self.h, None, sh))
        out = np.zeros(tuple(sh), np.float32)
        self.ref._check(self.ref.lib.ref_stepper_output(self.h, _ptr(out), sh))
        return out

    def close(self):
        if self.h:
            self.ref.lib.ref_stepper_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


class Oracle:
    """The plain-C restatement (double accumulation)."""

    def __init__(self):
        self.lib = C.CDLL(str(build_oracle()))
        self.lib.orc_optimal_fft_size.restype = C.c_int64

    def fill_random(self, count, seed):
        out = np.zeros(count, np.float32)
        self.lib.orc_fill_random_f32(_ptr(out), C.c_int64(count), C.c_uint64(seed))
        return out

    def random_weights(self, convs, seed):
        """convs: list of (fo, fin, kvol)."""
        fo = [c[0] for c in convs]
        fi = [c[1] for c in convs]
        k3 = [c[2] for c in convs]
        total = sum(a * b * c + a for a, b, c in convs)
        out = np.zeros(total, np.float32)
        self.lib.orc_random_weights_f32(_a64(fo), _a64(fi), _a64(k3), C.c_int64(len(convs)),
                                        C.c_uint64(seed), _ptr(out))
        return out

    def optimal_fft_size(self, n, profile):
        return int(self.lib.orc_optimal_fft_size(C.c_int64(n), C.c_int(profile)))

    def conv(self, x, w, bias, relu):
        x = np.ascontiguousarray(x, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        bias = np.ascontiguousarray(bias, np.float64)
        S, f = x.shape[:2]
        n = x.shape[2:]
        fo = w.shape[0]
        k = w.shape[2:]
        out = np.zeros((S, fo) + tuple(n[a] - k[a] + 1 for a in range(3)), np.float64)
        self.lib.orc_conv_direct(_ptr(x), C.c_int64(S), C.c_int64(f), _a64(n), _ptr(w),
                                 C.c_int64(fo), _a64(k), _ptr(bias), C.c_int(int(relu)), _ptr(out))
        return out

    def pool(self, fragments, x, p):
        x = np.ascontiguousarray(x, np.float32)
        S, f = x.shape[:2]
        n = x.shape[2:]
        no = tuple(n[a] // p[a] for a in range(3))
        P = int(np.prod(p)) if fragments else 1
        out = np.zeros((S * P, f) + no, np.float32)
        fn = self.lib.orc_mpf_pool if fragments else self.lib.orc_max_pool
        rc = fn(_ptr(x), C.c_int64(S), C.c_int64(f), _a64(n), _a64(p), _ptr(out))
        if rc:
            raise ValueError("pool: shape rule violated")
        return out

    def recombine(self, frag, windows, original_batch):
        frag = np.ascontiguousarray(frag, np.float32)
        S, f = frag.shape[:2]
        n = frag.shape[2:]
        stride = [1, 1, 1]
        for w in windows:
            stride = [stride[a] * w[a] for a in range(3)]
        out = np.zeros((original_batch, f) + tuple(stride[a] * n[a] for a in range(3)), np.float32)
        flat = [v for w in windows for v in w]
        rc = self.lib.orc_recombine(_ptr(frag), C.c_int64(S), C.c_int64(f), _a64(n),
                                    _a64(flat or [0]), C.c_int64(len(windows)),
                                    C.c_int64(original_batch), _ptr(out))
        if rc:
            raise ValueError("recombine: fragment batch mismatch")
        return out

    def pruned_fwd(self, img, pad):
        img = np.ascontiguousarray(img, np.float32)
        out = np.zeros((pad[0] // 2 + 1, pad[1], pad[2]), np.complex128)
        self.lib.orc_pruned_forward(_ptr(img), _a64(img.shape), _a64(pad), _ptr(out))
        return out

    def pruned_inv(self, spec, pad, crop):
        spec = np.ascontiguousarray(spec, np.complex128)
        out = np.zeros(tuple(crop), np.float64)
        self.lib.orc_pruned_inverse(_ptr(spec), _a64(pad), _a64(crop), _ptr(out))
        return out

    def batched_fwd(self, imgs, pad):
        imgs = np.ascontiguousarray(imgs, np.float32)
        b = imgs.shape[0]
        out = np.zeros((b, pad[2] // 2 + 1, pad[1], pad[0]), np.complex128)
        self.lib.orc_batched_forward(_ptr(imgs), C.c_int64(b), _a64(imgs.shape[1:]), _a64(pad),
                                     _ptr(out))
        return out

    def batched_inv(self, spec, pad, crop):
        spec = np.ascontiguousarray(spec, np.complex128)
        b = spec.shape[0]
        out = np.zeros((b,) + tuple(crop), np.float64)
        self.lib.orc_batched_inverse(_ptr(spec), C.c_int64(b), _a64(pad), _a64(crop), _ptr(out))
        return out

    def net_forward(self, layers, weights, x):
        """layers: list of ("conv", fo, (kx,ky,kz), relu) | ("mpf"|"plain", (px,py,pz))."""
        kind, ext, fo, relu = [], [], [], []
        for l in layers:
            if l[0] == "conv":
                kind.append(0)
                ext += list(l[2])
                fo.append(l[1])
                relu.append(int(l[3]))
            else:
                kind.append(1 if l[0] == "mpf" else 2)
                ext += list(l[1])
                fo.append(0)
                relu.append(0)
        x = np.ascontiguousarray(x, np.float32)
        S, f_in = x.shape[:2]
        e = x.shape[2:]
        # output shape via the shape rules
        n = list(e)
        s, f, strides = S, f_in, [1, 1, 1]
        for l in layers:
            if l[0] == "conv":
                n = [n[a] - l[2][a] + 1 for a in range(3)]
                f = l[1]
            else:
                p = l[1]
                if l[0] == "mpf":
                    strides = [strides[a] * p[a] for a in range(3)]
                n = [n[a] // p[a] for a in range(3)]
        out = np.zeros((S, f) + tuple(strides[a] * n[a] for a in range(3)), np.float64)
        w = np.ascontiguousarray(weights, np.float32)
        rc = self.lib.orc_net_forward(_a64(kind), _a64(ext), _a64(fo), _a64(relu),
                                      C.c_int64(len(layers)), _ptr(w), _ptr(x), C.c_int64(S),
                                      C.c_int64(f_in), _a64(e), _ptr(out))
        if rc:
            raise ValueError("net_forward: shape rule violated")
        return out


def rel_error(a, b) -> float:
    """oracle::rel_error (proj/tests/oracles.hpp:41-50): max|a-b| / max|b|."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / den if a.size else 0.0
