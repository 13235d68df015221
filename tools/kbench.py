"""Kernel-level timing probe (not the driver's bench): times single layers on
device-resident synthetic data with CUDA events on the library's stream.

    python tools/kbench.py [--which conv,mpf,direct,net] [--n 256]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1606_05688_b200 as v  # noqa: E402


def timed(ctx, fn, reps=3):
    s = torch.cuda.ExternalStream(ctx.stream())
    fn()
    ctx.sync()
    times = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        times.append(a.elapsed_time(b) * 1e-3)
    return min(times)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="conv,direct,mpf")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--T", type=int, default=0)
    ap.add_argument("--S", type=int, default=1)
    ap.add_argument("--net", default="n537")
    ap.add_argument("--extent", type=int, default=722)
    ap.add_argument("--tune", action="store_true")
    ap.add_argument("--k", type=int, default=7)
    ap.add_argument("--single-only", action="store_true")
    a = ap.parse_args()
    ctx = v.Context(0)
    res = {}
    g = torch.Generator(device="cuda").manual_seed(1)
    if "conv" in a.which:
        n = a.n
        x = torch.rand((a.S, 80, n, n, n), device="cuda", generator=g) * 2 - 1
        w = (torch.rand((80, 80, 5, 5, 5), device="cuda", generator=g) * 2 - 1) * 0.02
        b = torch.rand((80,), device="cuda", generator=g) * 0.2 - 0.1
        p = v.ConvLayerParams(w, b, "relu")
        ctx.profile(True)
        t = timed(ctx, lambda: v.conv_fft_staged(x, p, ctx))
        ks = ctx.kernel_stats()
        ctx.profile(False)
        no = n - 4
        res["conv_fft_80x80_k5_S%d_n%d" % (a.S, n)] = {
            "s": t, "vox_per_s": a.S * no ** 3 / t,
            "kernels": {k: round(s["seconds"] / s["launches"] * 1e3, 3) for k, s in ks.items()}}
        del x
    if "last" in a.which:
        # the 80 -> 3, k = 5 last layer of n537 at its bench fragment size
        n = a.n if a.n != 256 else 76
        S = a.S if a.S != 1 else 64
        x = torch.rand((S, 80, n, n, n), device="cuda", generator=g) * 2 - 1
        w = (torch.rand((3, 80, 5, 5, 5), device="cuda", generator=g) * 2 - 1) * 0.02
        b = torch.rand((3,), device="cuda", generator=g) * 0.2 - 0.1
        p = v.ConvLayerParams(w, b, "relu")
        for T in (12, 16, 24):
            ctx.profile(True)
            t = timed(ctx, lambda: v.conv_fft_tiled(x, p, T, tensor_cores=False, ctx=ctx))
            ks = ctx.kernel_stats()
            ctx.profile(False)
            res["last_80x3_k5_S%d_n%d_T%d" % (S, n, T)] = {
                "s": t, "kernels": {k: round(s["seconds"] / s["launches"] * 1e3, 3) for k, s in ks.items()}}
        del x
    if "tiles" in a.which:
        # one 80 -> 80 layer (kernel a.k) at tile size a.T: one CTA vs CTA-pair transforms
        n, kk = a.n, a.k
        x = torch.rand((a.S, 80, n, n, n), device="cuda", generator=g) * 2 - 1
        w = (torch.rand((80, 80, kk, kk, kk), device="cuda", generator=g) * 2 - 1) * 0.02
        b = torch.rand((80,), device="cuda", generator=g) * 0.2 - 0.1
        p = v.ConvLayerParams(w, b, "relu")
        for pair in ((False,) if a.single_only else (False, True)):
            ctx.profile(True)
            t = timed(ctx, lambda: v.conv_fft_tiled(x, p, a.T, tensor_cores=True, cta_pair=pair, ctx=ctx))
            ks = ctx.kernel_stats()
            ctx.profile(False)
            no = n - kk + 1
            res["tiles_80x80_k%d_S%d_n%d_T%d_%s" % (kk, a.S, n, a.T, "pair" if pair else "single")] = {
                "s": t, "ns_per_vox": t / (a.S * no ** 3) * 1e9,
                "kernels": {k2: round(s2["seconds"] * 1e3, 2) for k2, s2 in ks.items()}}
        del x
    if "direct" in a.which:
        n = 330
        x = torch.rand((1, 1, n, n, n), device="cuda", generator=g) * 2 - 1
        w = (torch.rand((80, 1, 4, 4, 4), device="cuda", generator=g) * 2 - 1) * 0.2
        b = torch.rand((80,), device="cuda", generator=g) * 0.2 - 0.1
        p = v.ConvLayerParams(w, b, "relu")
        t = timed(ctx, lambda: v.conv_direct(x, p, ctx))
        no = n - 3
        fl = 2.0 * 80 * 64 * no ** 3
        res["direct_1x80_k4_n330"] = {"s": t, "tflops": fl / t / 1e12}
    if "mpf" in a.which:
        n = 255
        x = torch.rand((1, 80, n, n, n), device="cuda", generator=g)
        t = timed(ctx, lambda: v.mpf_pool(x, (2, 2, 2), ctx))
        byt = 4.0 * 80 * (n ** 3 + 8 * 127 ** 3)
        res["mpf_80x255"] = {"s": t, "GBps": byt / t / 1e9}
    if "net" in a.which:
        from paper_1606_05688_b200.bundled_nets import NETS
        net = v.parse_network_spec(NETS[a.net])
        w = v.random_weights(net, 1)
        m = v.Model(net, w, ctx)
        e = a.extent
        algos = None
        if a.tune:
            m.tune(1, e)
            algos = ["direct"] + ["auto"] * (net.conv_count - 1)
        plan = m.plan_info(1, e, algos)
        x = torch.rand((1, 1, e, e, e), device="cuda", generator=g) * 2 - 1
        m.forward(x, cache_spectra=False, conv_algos=algos)
        ctx.sync()
        ctx.profile(True)
        t0 = time.perf_counter()
        _, rep = m.forward(x, cache_spectra=False, conv_algos=algos)
        ctx.sync()
        wall = time.perf_counter() - t0
        ks = ctx.kernel_stats()
        ctx.profile(False)
        res["net_%s_%d" % (a.net, e)] = {
            "seconds": rep.seconds, "wall": wall,
            "layers": [round(s, 4) for s in rep.layer_seconds],
            "planned": [round(l["seconds"], 4) for l in plan],
            "plan": [(l.get("algo", "pool"), l.get("T", 0)) for l in plan],
            "kernels": {k: {"s": round(s["seconds"], 4), "n": s["launches"],
                            "TFLOPs": round(s["flops"] / s["seconds"] / 1e12, 1) if s["flops"] else None,
                            "GBps": round(s["bytes"] / s["seconds"] / 1e9) if s["bytes"] else None}
                        for k, s in ks.items()}}
        m.close()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
