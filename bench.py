#!/usr/bin/env python
"""n537 sliding-window 3D ConvNet inference throughput on B200 (output voxels/s).

One step = one device-resident forward of the bundled n537 network over one
cubic input patch (synthetic: random_weights(net, 1) and the reference's
fill_random generator), every pool as MPF, fragments recombined into the dense
output.  The patch is the largest admissible extent (e = 2 mod 8) whose
planned peak fits the HBM budget, unless --extent.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (weak scaling: one patch per GPU per step)

Prints ONE JSON line (rank 0).  `value` is device-timed with inputs resident
in HBM; `e2e` goes through the public API with pinned host buffers
(H2D + forward + D2H inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

NET = "n537"
# smallest admissible cubic patch per bundled net: the CPU
# reference runs there
SMALLEST = {"n337": 92, "n537": 170, "n726": 120, "n926": 158}
# ncu dram__bytes_read.sum + dram__bytes_write.sum / algorithmic bytes of one
# cgemm_q_kernel<80, 1> launch (kbench 80 -> 80 k5, S = 64, n = 85, T = 32, 1728
# rows: 24.14 + 19.22 GB against 8 * 17408 * (2 * 1728 * 80 + 80 * 80) B = 39.39 GB),
# profiles/r2/h3_layer_full.txt
TRAFFIC_RATIO = {"cgemm": round((24.143 + 19.217) / 39.394, 3)}
TRAFFIC_SOURCE = "profiles/r2/h3_layer_full.txt"
FFMA_FALLBACK_TFLOPS = 74.4  # 148 SM x 128 x 2 x 1.965 GHz (nominal), used only if measurement fails


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--net", default=NET, choices=["n337", "n537", "n726", "n926"],
                    help="bundled network (the headline metric is n537)")
    ap.add_argument("--extent", type=int, default=0, help="cubic input extent (0: largest that fits)")
    ap.add_argument("--budget-gb", type=float, default=0.0)
    ap.add_argument("--cache-spectra", type=int, default=0,
                    help="1: reuse kernel spectra across steps (weights fixed); 0: recompute per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--quick", action="store_true", help="small extent (profiling / smoke)")
    ap.add_argument("--no-tune", action="store_true", help="modelled (not measured) layer planning")
    ap.add_argument("--stub", action="store_true", help=argparse.SUPPRESS)  # CPU test of the N > 1 launch path
    ap.add_argument("--ref-planner", action="store_true",
                    help="--impl reference: also time one forward with the reference planner's own plan")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def bench_seed(seed, e):
    """cli.cpp:261: the bench input seed for extent e."""
    return (seed ^ ((0x9E3779B97F4A7C15 * e) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text()), "measured"
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def pick_extent(model, budget_bytes, fov, hi=2048, algos=None, fout=3):
    """Largest admissible extent (one that propagates through every MPF) whose plan fits."""
    best = None
    e = hi
    while e >= fov:
        need = model.plan_bytes(1, e, algos)
        if 0 < need:
            # device input + dense output of the timed run live outside the plan
            extra = 4 * (e ** 3) + 4 * fout * (e - fov + 1) ** 3
            if need + extra <= budget_bytes:
                best = e
                break
        e -= 1
    return best


def choose_patch(model, net, fov, budget_bytes, tuned, extent=0, quick=False):
    """(extent, conv algos) of the bench step: the largest admissible patch whose
    plan fits the budget, or -- with measured layer costs -- the (patch,
    first-layer algorithm) pair of highest estimated throughput among the
    largest few fitting patches: a direct first layer fuses with the MPF after
    it (its full-resolution output never exists) and so admits a larger patch
    than an FFT one.  Also used by the GPU parity tests to run the bench's plan."""
    if extent:
        return extent, None
    if quick:
        return 258, None
    nconv = sum(1 for l in net.layers if l[0] == "conv")
    step = 1  # admissible extents repeat with the MPF stride product
    for l in net.layers:
        if l[0] == "pool":
            step *= l[1][0]
    if not tuned:
        return pick_extent(model, budget_bytes, fov, fout=net.features_out), None
    best = None
    for algos in (None, ["direct"] + ["auto"] * (nconv - 1)):
        emax = pick_extent(model, budget_bytes, fov, algos=algos, fout=net.features_out)
        if emax is None:
            continue
        for e in range(emax, max(fov, emax - step * 12) - 1, -step):
            est = sum(l["seconds"] for l in model.plan_info(1, e, algos))
            score = (e - fov + 1) ** 3 / est if est > 0 else 0
            if best is None or score > best[0]:
                best = (score, e, algos)
    return (best[1], best[2]) if best else (None, None)


def layer_roofline(net_layers, e, fov, peak_fp32, peak_hbm, per_layer=None):
    """sum over layers of max(F_l / P_fp32, B_l / P_hbm) with
    F_fft = 7.5 S (f+f') N^3 log2 N + 2.5 f f' N log2 N (k^2 + kN + N^2) + 8 S f f' #w,
    F_dir = 2 S f f' n'^3 k^3 (the cheaper conv per layer), MPF bytes
    4 S f (n^3 + p^3 floor(n/p)^3); N = optimal_fft_size(n, device profile)."""
    import math
    from paper_1606_05688_b200 import optimal_fft_size
    S, f, n = 1, 1, e
    total = 0.0
    for l in net_layers:
        if l[0] == "conv":
            fo, k = l[1], l[2][0]
            no = n - k + 1
            N = optimal_fft_size(n, "device")
            lg = math.log2(N)
            nw = N * N * (N // 2 + 1)
            F_fft = 7.5 * S * (f + fo) * N ** 3 * lg + 2.5 * f * fo * N * lg * (k * k + k * N + N * N) \
                + 8.0 * S * f * fo * nw
            F_dir = 2.0 * S * f * fo * no ** 3 * k ** 3
            B = 4.0 * (S * f * n ** 3 + S * fo * no ** 3 + f * fo * k ** 3 + fo)
            t = max(min(F_fft, F_dir) / (peak_fp32 * 1e12), B / (peak_hbm * 1e9))
            total += t
            if per_layer is not None:
                per_layer.append(t)
            f, n = fo, no
        else:
            p = l[1][0]
            m = n // p
            B = 4.0 * S * f * (n ** 3 + p ** 3 * m ** 3)
            total += B / (peak_hbm * 1e9)
            if per_layer is not None:
                per_layer.append(B / (peak_hbm * 1e9))
            S *= p ** 3
            n = m
    return total


def bundled_nets():
    """NETS / FOV of paper_1606_05688_b200/bundled_nets.py, loaded by file path:
    importing the package would map libvxg.so into the process, and the
    reference arm must run without any of the product's native code."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_vxg_bundled_nets", ROOT / "paper_1606_05688_b200" / "bundled_nets.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.NETS, mod.FOV


def reference_steps(ref, net_text, e, plan, warmup, steps, nlayers):
    """The reference's execute_plan (host-only plan: run_prefix + recombine,
    proj/include/voxin/execute.hpp:147-226, 388-402) run one layer per step
    (oracle/ref_shim.cpp ref_stepper_*; bit-identical to execute_plan,
    tests/test_oracle.py).  A step is one layer of a forward, forwards follow
    each other from the same input; `warmup` untimed steps, then `steps` timed
    ones, extended until every layer was timed at least once.  Forward time =
    sum over layers of the layer's mean timed seconds."""
    st = ref.stepper(net_text, e, 1, bench_seed(1, e), plan=plan, conv_kind=3, nlayers=nlayers)
    for _ in range(warmup):
        st.step()
    per_layer = {}
    timed = []
    while len(timed) < steps or len(per_layer) < nlayers:
        li, sec, _ = st.step()
        per_layer.setdefault(li, []).append(sec)
        timed.append(sec)
    fwd = sum(sum(v) / len(v) for v in per_layer.values())
    kinds = st.kinds
    st.close()
    return {"forward_seconds": fwd, "timed_steps": len(timed), "step_seconds": timed,
            "layer_seconds": {int(k): sum(v) / len(v) for k, v in sorted(per_layer.items())}, "kinds": kinds}


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    compiled from the unmodified sources) on all host cores, through its
    execute_plan (layer-stepped) with conv forced to fft_task_parallel (the
    fastest measured reference primitive), every pool MPF; then
    one forward with the reference planner's own plan (optimize_plan) for
    context.  No product code is imported."""
    if ws > 1 and rank != 0:
        return
    from oracle.refbind import Ref
    NETS, FOV = bundled_nets()
    ref = Ref(workers=0)
    e = SMALLEST[args.net]  # smallest admissible patch: a forward the CPU path finishes in bounded time
    text = NETS[args.net]
    nlayers = sum(1 for l in text.splitlines() if l.startswith(("conv", "pool")))
    vox = (e - FOV[args.net] + 1) ** 3
    main_run = reference_steps(ref, text, e, "forced", args.warmup, args.steps, nlayers)
    value = vox / main_run["forward_seconds"]
    # the reference planner's own plan (fft_data_parallel everywhere for n537:
    # ~330 s per forward on 16 cores) only on request, to keep the arm to minutes
    planner_run = reference_steps(ref, text, e, "planner", 0, nlayers, nlayers) if args.ref_planner else None
    steps_s = main_run["step_seconds"]
    line = {
        "impl": "reference", "metric": f"output voxels/sec, {args.net} 3D ConvNet sliding-window inference",
        "value": value, "unit": "voxels/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(steps_s) / len(steps_s), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.net} full forward, input {e}^3 -> dense {e - FOV[args.net] + 1}^3, "
                               "all pools MPF, conv fft_task_parallel (reference execute_plan, host-only plan)",
                   "net": args.net, "extent": e,
                   "step": "one layer of execute_plan's host-only path (the forward runs layer by layer "
                           "across steps; forward time = sum of mean layer times)",
                   "timed_steps_run": main_run["timed_steps"]},
        "cpu_baseline": {"value": value, "unit": "voxels/s", "cores": ref.workers, "kind": "reference",
                         "sample": f"{args.net} at {e}^3: {main_run['timed_steps']} timed layer steps of "
                                   "the reference execute_plan (fft_task_parallel, MPF), after "
                                   f"{args.warmup} warm-up steps"},
        "e2e": {"value": value, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "forward_seconds": main_run["forward_seconds"],
        "layer_seconds": main_run["layer_seconds"],
    }
    if planner_run:
        line["reference_planner_plan"] = {
            "kinds": planner_run["kinds"], "forward_seconds": planner_run["forward_seconds"],
            "value": vox / planner_run["forward_seconds"],
            "note": f"the reference's optimize_plan (HostModel, workers = cores) at extent {e}, one forward"}
    print(json.dumps(line), flush=True)


def cpu_baseline(args):
    """Reference CPU path on the box's host cores (rank 0, N = 1): one full
    forward (one step per layer) of the reference's execute_plan at the
    smallest admissible patch through oracle/_ref (no product code)."""
    try:
        from oracle.refbind import Ref
        NETS, FOV = bundled_nets()
        ref = Ref(workers=0)
    except Exception as ex:  # pragma: no cover
        return {"value": None, "unit": "voxels/s", "cores": 0, "kind": "reference",
                "sample": f"unavailable: {ex}"}
    e = SMALLEST[args.net]
    text = NETS[args.net]
    nlayers = sum(1 for l in text.splitlines() if l.startswith(("conv", "pool")))
    run = reference_steps(ref, text, e, "forced", 0, nlayers, nlayers)
    vox = (e - FOV[args.net] + 1) ** 3
    return {"value": vox / run["forward_seconds"], "unit": "voxels/s", "cores": ref.workers, "kind": "reference",
            "seconds": run["forward_seconds"],
            "sample": f"one full {args.net} forward at its smallest admissible patch {e}^3 -> dense "
                      f"{e - FOV[args.net] + 1}^3: the reference's execute_plan (oracle/_ref, unmodified "
                      "sources), conv fft_task_parallel, pools MPF, recombined; fp32"}


def self_launch(args):
    """`--gpus N` (N > 1) without a torch.distributed environment: re-run this
    script under torch.distributed.run with N ranks on this node (rendezvous on
    127.0.0.1), so a bare `python bench.py --gpus 8` measures 8 GPUs."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_stub(args, ws, rank):
    """--stub (CPU tests of the N > 1 launch path): the bench's distributed
    skeleton -- self-launch, barrier, max-over-ranks timing, whole-job value --
    over gloo with a numpy stand-in step (a translation-equivariant box filter
    on this rank's own tile); no GPU, no product code."""
    import numpy as np
    import torch
    import torch.distributed as dist
    if ws > 1:
        dist.init_process_group("gloo")
    e, fov = 48, 9
    x = np.random.default_rng(rank).standard_normal((e, e, e)).astype(np.float32)

    def step():
        c = x.cumsum(0).cumsum(1).cumsum(2)
        return float(c[-1, -1, -1])

    for _ in range(args.warmup):
        step()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    elapsed = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([elapsed], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
        dist.barrier()
    voxels = (e - fov + 1) ** 3
    if rank == 0:
        print(json.dumps({"metric": "stub", "value": ws * args.steps * voxels / elapsed, "unit": "voxels/s",
                          "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": 1e3 * elapsed / args.steps, "scaling": "weak", "stub": True,
                          "voxels_per_rank_step": voxels, "elapsed_max_over_ranks": elapsed}), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.stub:
        run_stub(args, ws, rank)
        return
    if ws != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={ws}")

    import numpy as np
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1606_05688_b200 as v
    from paper_1606_05688_b200.bundled_nets import FOV, NETS

    net = v.parse_network_spec(NETS[args.net])
    fov = FOV[args.net]
    weights = v.random_weights(net, 1)
    peaks, peaks_src = measured_peaks()

    budget = int(args.budget_gb * 1e9) if args.budget_gb > 0 else 0
    ctx = v.Context(local, budget)
    model = v.Model(net, weights, ctx)
    budget_bytes = ctx.memory()["budget"]

    def choose(tuned):
        return choose_patch(model, net, fov, budget_bytes, tuned, args.extent, args.quick)

    e, algos = choose(False)
    if e is None:
        raise SystemExit("no admissible extent fits the HBM budget")
    # measured-time layer planner: candidate tile sizes / direct timed on samples
    # of each conv layer (outside the timed region), then the patch re-picked
    t_tune = time.perf_counter()
    if not args.no_tune:
        model.tune(1, e)
        e, algos = choose(True)
    if ws > 1:
        # every rank processes rank 0's patch shape (its own tile of the volume),
        # so value = ws * voxels is exact even if per-rank timings differ
        pick = [e, algos]
        dist.broadcast_object_list(pick, src=0)
        e, algos = pick
    t_tune = time.perf_counter() - t_tune
    plan = model.plan_info(1, e, algos)
    dense = e - fov + 1
    voxels = dense ** 3

    # synthetic input (the reference's generator; rank-specific seed = another tile)
    x_host = v.fill_random((1, 1, e, e, e), bench_seed(1 + rank, e))
    x_pin = torch.from_numpy(x_host).pin_memory()
    x_dev = x_pin.cuda()
    fout = net.features_out
    out_dev = torch.empty((1, fout, dense, dense, dense), dtype=torch.float32, device="cuda")
    stream = torch.cuda.ExternalStream(ctx.stream())
    cache = bool(args.cache_spectra)

    last = {}

    def step():
        last["rep"] = model.forward(x_dev, out=out_dev, conv_algos=algos, cache_spectra=cache)[1]

    for _ in range(args.warmup):
        step()
    ctx.sync()

    ffma_peak = ctx.bench_ffma()
    if not (ffma_peak > 1.0):
        ffma_peak = FFMA_FALLBACK_TFLOPS

    # ---- timed region (device events on the library stream) ----
    clocks = ClockSampler(local)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.sync()
    clocks.start()
    ctx.profile(True)
    launches0 = ctx.launches
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    ev1.synchronize()
    ctx.sync()
    elapsed = ev0.elapsed_time(ev1) * 1e-3
    launches = ctx.launches - launches0
    kstats = ctx.kernel_stats()
    ctx.profile(False)
    clk = clocks.stop()
    torch.cuda.synchronize()
    if ws > 1:
        t = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
        dist.barrier()
    value = ws * args.steps * voxels / elapsed

    # ---- e2e through the public API, host buffers ----
    out_host = torch.empty((1, fout, dense, dense, dense), dtype=torch.float32).pin_memory()
    xin = x_pin.numpy()
    oh = out_host.numpy()
    # warm the streaming path itself: its double buffers change the forward's
    # arena size, and the pool maps a block of the new size only once
    model.forward_many([xin] * 2, outputs=[oh] * 2, conv_algos=algos, cache_spectra=cache)
    if ws > 1:
        dist.barrier()
    # the streaming API (the tiler's path): every step uploads its patch and
    # downloads its result; copies of neighbouring steps overlap the forwards
    t0 = time.perf_counter()
    model.forward_many([xin] * args.e2e_steps, outputs=[oh] * args.e2e_steps, conv_algos=algos,
                       cache_spectra=cache)
    e2e_t = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([e2e_t], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e = {"value": ws * args.e2e_steps * voxels / e2e_t, "unit": "voxels/s",
           "h2d_bytes_per_step": int(x_host.nbytes), "d2h_bytes_per_step": int(oh.nbytes),
           "steps": args.e2e_steps,
           "api": "vxg_model_forward_many (pinned host patches, double-buffered uploads/downloads "
                  "overlapping the forwards) via paper_1606_05688_b200.Model.forward_many"}

    # ---- roofline of the dominant kernel (live CUDA-event times) ----
    kernels = {}
    total_k = sum(s["seconds"] for s in kstats.values()) or 1.0
    for name, s in kstats.items():
        d = {"launches": s["launches"], "seconds": s["seconds"], "share": s["seconds"] / elapsed}
        if s["flops"] > 0:
            d["tflops"] = s["flops"] / s["seconds"] / 1e12
        if s["bytes"] > 0:
            d["gbps"] = s["bytes"] / s["seconds"] / 1e9
        kernels[name] = d
    dom = max(kstats, key=lambda k: kstats[k]["seconds"])
    tc_used = os.environ.get("VXG_NO_TC", "0") in ("", "0")
    ds = kstats[dom]
    if ds["flops"] > 0 and dom == "cgemm" and tc_used:
        # tcgen05: a tf32 MMA for a_hi*b_hi plus one kind::f16 MMA (K = 16, same
        # time as a K = 8 tf32 MMA) for both bf16 correction terms -- 2 tf32-MMA
        # equivalents per real product (VXG_Q_3TF32=1: the 3xTF32 split, 3) -- so
        # the algorithmic-fp32 ceiling is the tf32 peak (1/2 of the measured dense
        # bf16 peak) / 2 (or / 3).  The contraction also moves X + Y + W through
        # HBM: report against whichever bound is slower for its per-launch work.
        tflops = ds["flops"] / ds["seconds"] / 1e12
        gbps = ds["bytes"] / ds["seconds"] / 1e9
        # sustained figure: the contraction runs inside a seconds-long step
        tkey = "bf16_tflops_sustained" if "bf16_tflops_sustained" in peaks else "bf16_tflops"
        split = 3.0 if os.environ.get("VXG_Q_3TF32") else 2.0
        tpeak = peaks.get(tkey, 1395.3) / 2.0 / split
        t_tensor = ds["flops"] / (tpeak * 1e12)
        t_hbm = ds["bytes"] / (peaks["hbm_gbs"] * 1e9)
        if t_hbm >= t_tensor:
            roof = {"kernel": dom, "bound": "hbm", "achieved": gbps, "peak": peaks["hbm_gbs"],
                    "unit": "GB/s", "frac": gbps / peaks["hbm_gbs"], "peak_source": peaks_src,
                    "tensor_frac": tflops / tpeak}
        else:
            roof = {"kernel": dom, "bound": "tensor", "achieved": tflops, "peak": tpeak,
                    "unit": "TFLOP/s", "frac": tflops / tpeak,
                    "peak_source": f"MEASURED_PEAKS.json {tkey} ({peaks_src}) / 2 (tf32) / {split:g} (MMAs per product)",
                    "hbm_frac": gbps / peaks["hbm_gbs"]}
        roof["tensor_peak_tflops"] = tpeak
        roof["vs_fp32_ffma_peak"] = tflops / ffma_peak
    elif ds["flops"] > 0:
        ach = ds["flops"] / ds["seconds"] / 1e12
        roof = {"kernel": dom, "bound": "fp32", "achieved": ach, "peak": ffma_peak,
                "unit": "TFLOP/s", "frac": ach / ffma_peak,
                "peak_source": "measured FFMA microbenchmark (vxg_bench_ffma; MEASURED_PEAKS.json "
                               "has no fp32 figure)"}
    else:
        ach = ds["bytes"] / ds["seconds"] / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": ach / peaks["hbm_gbs"], "peak_source": peaks_src}
    # DRAM traffic / algorithmic bytes of the dominant kernel from the committed
    # ncu --set full capture (TRAFFIC_SOURCE), applied per launch
    ratio = TRAFFIC_RATIO.get(dom)
    roof["traffic"] = ratio * ds["bytes"] / ds["launches"] if ratio else None
    roof["traffic_source"] = ("ncu dram__bytes_read.sum + dram__bytes_write.sum / algorithmic bytes = "
                              f"{ratio} ({TRAFFIC_SOURCE})") if ratio else None
    roof["per_launch"] = {"flops": ds["flops"] / ds["launches"], "bytes": ds["bytes"] / ds["launches"],
                          "seconds": ds["seconds"] / ds["launches"]}
    roof_l = []
    t_roof = layer_roofline(net.layers, e, fov, ffma_peak, peaks["hbm_gbs"], roof_l)
    step_s = elapsed / args.steps
    meas_l = list(last["rep"].layer_seconds)
    per_layer = [{"layer": i, "kind": ("conv" if l[0] == "conv" else "pool"),
                  "plan": (f"{p.get('algo')}/T{p.get('T')}" if p["kind"] == "conv" else "mpf"),
                  "measured_s": round(meas_l[i], 5) if i < len(meas_l) else None,
                  "roofline_s": round(roof_l[i], 5)}
                 for i, (l, p) in enumerate(zip(net.layers, plan))]
    net_roof = {"seconds": t_roof, "step_seconds": step_s, "frac": t_roof / step_s,
                "per_layer": per_layer,
                "definition": "SURVEY 8(d): sum_l max(F_l/P_fp32, B_l/P_hbm), F = cheaper of "
                              "whole-image pruned FFT and direct, P_fp32 = measured FFMA peak"}

    line = {
        "metric": f"output voxels/sec, {args.net} 3D ConvNet sliding-window inference",
        "value": value, "unit": "voxels/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * step_s, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.net} full forward per GPU, input patch {e}^3 -> dense {net.features_out}x{dense}^3 "
                               "(largest admissible patch fitting the HBM budget)",
                   "net": args.net, "extent": e, "dense_out": dense, "global_batch": ws,
                   "parallelism": f"independent halo patches x{ws}",
                   "kernel_spectra": "cached across steps" if cache else "recomputed every step",
                   "planner": ("modelled" if args.no_tune else
                               (f"measured costs replayed from {os.environ['VXG_TUNE_FILE']}"
                                if os.environ.get("VXG_TUNE_FILE") else
                                f"measured (vxg_model_tune, {t_tune:.1f} s before the timed region)")),
                   "planned_step_s": round(sum(l["seconds"] for l in plan), 4),
                   "layers": " ".join(
                       (f"L{l['layer']}:{l['algo']}" + (f"/T{l['T']}" + (("/tc" if l.get('tc_tiles') != "pair" else "/tcp") if l['tc'] else "/ffma")
                                                          if l['algo'] == 'fft' else ""))
                       if l["kind"] == "conv" else f"L{l['layer']}:mpf" for l in plan),
                   "l2": "inputs and activations >> 126 MB L2 (no flush needed)"},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
        "roofline": roof,
        "layer_roofline": net_roof,
        "kernels": kernels,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    model.close()
    ctx.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
