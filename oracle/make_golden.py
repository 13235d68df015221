"""TEST INFRASTRUCTURE: generate tests/golden/*.npz by running the UNMODIFIED
reference (oracle/_ref/libvoxref.so, compiled from /root/reference/proj by
oracle/build_ref.sh) on seeded inputs.  Run here (the reference sources do not
exist on the GPU box); the fixtures are committed.

    python oracle/make_golden.py [--nets]     # --nets adds the bundled-net runs (minutes)

Every random array is produced by the reference's own generators
(fill_random = cli.cpp:78-84, random_weights = execute.hpp:50-73) so a test
can regenerate big inputs from the stored seed instead of storing them.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle.refbind import Ref  # noqa: E402

REF_NETS = Path("/root/reference/proj/nets")
GOLD = Path(__file__).resolve().parent.parent / "tests" / "golden"

# toy nets used by the reference's own tests (acceptance.cpp:132-137, and the
# 3-MPF chain the survey verified against the sliding-window oracle)
TOY_NETS = {
    "c3": "input 1\nconv 4 3 relu\npool 2 mpf\nconv 4 3 relu\npool 2 mpf\nconv 2 3\n",
    "mpf3": "input 1\nconv 3 2 relu\npool 2 mpf\nconv 3 2 relu\npool 2 mpf\nconv 3 2 relu\n"
            "pool 2 mpf\nconv 2 2\n",
    "aniso": "input 2\nconv 3 3 2 3 relu\npool 1 2 2 mpf\nconv 2 2 3 2\n",
}


def parse_layers(text):
    """Minimal reader of the .net grammar (netspec.hpp:89-99) for test bookkeeping."""
    fin, layers = None, []
    for line in text.splitlines():
        tok = line.split("#")[0].split()
        if not tok:
            continue
        if tok[0] == "input":
            fin = int(tok[1])
        elif tok[0] == "conv":
            relu = tok[-1] == "relu"
            nums = [int(t) for t in (tok[1:-1] if relu else tok[1:])]
            k = tuple(nums[1:]) * 3 if len(nums) == 2 else tuple(nums[1:])
            layers.append(("conv", nums[0], k, relu))
        elif tok[0] == "pool":
            nums = [int(t) for t in tok[1:] if t not in ("mpf", "plain", "auto")]
            p = tuple(nums) * 3 if len(nums) == 1 else tuple(nums)
            layers.append(("mpf", p))
    return fin, layers


def weight_count(fin, layers):
    f, total = fin, 0
    for l in layers:
        if l[0] == "conv":
            total += l[1] * f * int(np.prod(l[2])) + l[1]
            f = l[1]
    return total


def out_shape(fin, layers, S, e):
    n, f, st = list(e), fin, [1, 1, 1]
    for l in layers:
        if l[0] == "conv":
            n = [n[a] - l[2][a] + 1 for a in range(3)]
            f = l[1]
        else:
            st = [st[a] * l[1][a] for a in range(3)]
            n = [n[a] // l[1][a] for a in range(3)]
    return (S, f) + tuple(st[a] * n[a] for a in range(3))


def bench_seed(seed, e):
    """cli.cpp:261: fill_random seed for extent e."""
    return (seed ^ ((0x9E3779B97F4A7C15 * e) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF


def gen_basic(ref: Ref):
    g = {}
    # generators (pinned so tests can regenerate big inputs from seeds)
    g["fill_random_seed7_f32"] = ref.fill_random(4096, 7, 32)
    g["fill_random_seed7_f64"] = ref.fill_random(4096, 7, 64)
    for name, text in TOY_NETS.items():
        fin, layers = parse_layers(text)
        g[f"weights_{name}_seed11"] = ref.random_weights(text, 11, weight_count(fin, layers), 32)
    # padded sizes (fft_test.cpp:12-46 and the survey's device sizes)
    ns = np.arange(1, 700, dtype=np.int64)
    g["fft_size_n"] = ns
    g["fft_size_host"] = np.array([ref.optimal_fft_size(n, 0) for n in ns], np.int64)
    g["fft_size_dev"] = np.array([ref.optimal_fft_size(n, 1) for n in ns], np.int64)
    g["fft_size_any"] = np.array([ref.optimal_fft_size(n, 2) for n in ns], np.int64)
    np.savez_compressed(GOLD / "basic.npz", **g)


def gen_pools(ref: Ref):
    g = {}
    rng_seed = 100
    # pinned lines (layers_test.cpp:48-132)
    g["pin_pool_in"] = np.array([1, 5, 3, 2, 9, 0], np.float32).reshape(1, 1, 1, 1, 6)
    g["pin_pool_out"] = ref.pool(False, g["pin_pool_in"], (1, 1, 2), 32)
    g["pin_mpf_in"] = np.array([1, 5, 3, 2, 9], np.float32).reshape(1, 1, 1, 1, 5)
    g["pin_mpf_out"] = ref.pool(True, g["pin_mpf_in"], (1, 1, 2), 32)
    cases = [
        ("mpf", (1, 2, (5, 5, 5)), (2, 2, 2)),
        ("mpf", (2, 3, (7, 9, 5)), (2, 2, 2)),
        ("mpf", (1, 2, (8, 5, 11)), (3, 2, 3)),
        ("mpf", (3, 1, (6, 7, 9)), (1, 2, 5)),
        ("mpf", (1, 4, (17, 17, 17)), (2, 2, 2)),
        ("plain", (2, 2, (6, 6, 6)), (2, 2, 2)),
        ("plain", (1, 3, (9, 4, 10)), (3, 2, 5)),
        ("plain", (1, 2, (5, 5, 5)), (1, 1, 1)),
    ]
    for i, (kind, (S, f, n), p) in enumerate(cases):
        x = ref.fill_random(S * f * int(np.prod(n)), rng_seed + i, 32).reshape((S, f) + n)
        g[f"case{i}_kind"] = np.array(1 if kind == "mpf" else 0)
        g[f"case{i}_p"] = np.array(p, np.int64)
        g[f"case{i}_in"] = x
        g[f"case{i}_out"] = ref.pool(kind == "mpf", x, p, 32)
    g["ncases"] = np.array(len(cases))
    # recombination (layers_test.cpp:113-132 pinned, plus multi-window)
    g["pin_rec_in"] = np.array([1, 2, 3, 4], np.float32).reshape(2, 1, 1, 1, 2)
    g["pin_rec_out"] = ref.recombine(g["pin_rec_in"], [(1, 1, 2)], 1, 32)
    rcases = [
        ([(2, 2, 2)], 1, 3, (3, 4, 2)),
        ([(2, 2, 2), (2, 2, 2)], 2, 2, (2, 3, 3)),
        ([(2, 2, 2), (3, 1, 2), (1, 2, 2)], 1, 1, (2, 2, 3)),
        ([(2, 2, 2), (2, 2, 2), (2, 2, 2)], 1, 3, (4, 4, 4)),
    ]
    for i, (wins, S0, f, n) in enumerate(rcases):
        alpha = int(np.prod([np.prod(w) for w in wins]))
        x = ref.fill_random(S0 * alpha * f * int(np.prod(n)), 200 + i, 32).reshape(
            (S0 * alpha, f) + n)
        g[f"rec{i}_win"] = np.array(wins, np.int64)
        g[f"rec{i}_S0"] = np.array(S0)
        g[f"rec{i}_in"] = x
        g[f"rec{i}_out"] = ref.recombine(x, wins, S0, 32)
    g["nrec"] = np.array(len(rcases))
    np.savez_compressed(GOLD / "pools.npz", **g)


def gen_fft(ref: Ref):
    g = {}
    # fft_test.cpp:48-206 case list plus device-sized pads
    cases = [((4, 5, 6), (4, 5, 6)), ((3, 3, 3), (4, 4, 4)), ((2, 2, 2), (6, 6, 6)),
             ((5, 1, 4), (6, 2, 4)), ((5, 4, 3), (6, 5, 4)), ((9, 7, 12), (10, 7, 12)),
             ((5, 5, 5), (27, 25, 21)), ((30, 17, 9), (30, 18, 10))]
    for i, (n, pad) in enumerate(cases):
        x = ref.fill_random(int(np.prod(n)), 300 + i, 32).reshape(n)
        g[f"p{i}_n"] = np.array(n, np.int64)
        g[f"p{i}_pad"] = np.array(pad, np.int64)
        g[f"p{i}_in"] = x
        g[f"p{i}_nested"] = ref.pruned_fwd(x, pad, 64)
        g[f"p{i}_inv"] = ref.pruned_inv(g[f"p{i}_nested"], pad, n, 64)
        xb = ref.fill_random(3 * int(np.prod(n)), 400 + i, 32).reshape((3,) + n)
        g[f"p{i}_bin"] = xb
        g[f"p{i}_batched"] = ref.batched_fwd(xb, pad, 64)
        g[f"p{i}_binv"] = ref.batched_inv(g[f"p{i}_batched"], pad, n, 64)
    g["ncases"] = np.array(len(cases))
    np.savez_compressed(GOLD / "fft.npz", **g)


def gen_conv(ref: Ref):
    g = {}
    # layers_test.cpp:162-364 case shapes, plus the net-layer shapes at small n
    cases = [
        (1, 1, (6, 6, 6), 1, (1, 1, 1), False),
        (2, 3, (9, 8, 7), 4, (3, 2, 3), True),
        (1, 1, (12, 12, 12), 8, (4, 4, 4), True),
        (1, 2, (5, 6, 7), 3, (5, 6, 7), False),          # k = n
        (3, 5, (10, 11, 9), 6, (2, 3, 4), True),
        (1, 16, (14, 14, 14), 16, (5, 5, 5), True),
        (2, 80, (11, 11, 11), 80, (5, 5, 5), True),       # the 80->80 k5 layer at small n
        (1, 80, (13, 13, 13), 3, (5, 5, 5), True),        # the 80->3 output layer
        (1, 7, (20, 9, 16), 5, (7, 3, 9), True),
    ]
    for i, (S, f, n, fo, k, relu) in enumerate(cases):
        x = ref.fill_random(S * f * int(np.prod(n)), 500 + i, 32).reshape((S, f) + n)
        w = ref.fill_random(fo * f * int(np.prod(k)), 600 + i, 32).reshape((fo, f) + k)
        w *= np.float32(np.sqrt(3.0 / (f * np.prod(k))))
        b = ref.fill_random(fo, 700 + i, 32) * np.float32(0.1)
        g[f"c{i}_in"] = x
        g[f"c{i}_w"] = w
        g[f"c{i}_b"] = b
        g[f"c{i}_relu"] = np.array(int(relu))
        g[f"c{i}_out64"] = ref.conv(0, x, w, b, relu, 64)        # direct, fp64
        g[f"c{i}_fft32"] = ref.conv(3, x, w, b, relu, 32)        # task-parallel fft, fp32
    g["ncases"] = np.array(len(cases))
    np.savez_compressed(GOLD / "conv.npz", **g)


def gen_nets(ref: Ref, bundled: bool):
    meta = {}
    g = {}
    runs = [(name, text, e) for name, text, e in [
        ("c3", TOY_NETS["c3"], (21, 21, 21)),
        ("mpf3", TOY_NETS["mpf3"], (38, 38, 38)),
        ("aniso", TOY_NETS["aniso"], (9, 12, 13)),
    ]]
    if bundled:
        # the smallest admissible cubic extent of each bundled net
        for name, e in [("n337", 92), ("n726", 120), ("n926", 158), ("n537", 170)]:
            runs.append((name, (REF_NETS / f"{name}.net").read_text(), (e, e, e)))
    for name, text, e in runs:
        fin, layers = parse_layers(text)
        wseed = 1
        iseed = bench_seed(1, e[0])
        x = ref.fill_random(fin * int(np.prod(e)), iseed, 32).reshape((1, fin) + e)
        shape = out_shape(fin, layers, 1, e)
        t0 = time.time()
        out, secs = ref.net_forward(text, wseed, x, conv_kind=3, mpf=True, prec=64, out_shape=shape)
        print(f"{name} @ {e}: out {shape} in {time.time() - t0:.1f}s", flush=True)
        g[f"{name}_out64"] = out
        meta[name] = {"text": text, "extent": list(e), "wseed": wseed, "iseed": iseed,
                      "out_shape": list(shape), "ref_seconds_fp64": secs}
    suffix = "_bundled" if bundled else ""
    np.savez_compressed(GOLD / f"nets{suffix}.npz", **g)
    (GOLD / f"nets{suffix}.json").write_text(json.dumps(meta, indent=1))


def gen_shapes(ref: Ref):
    meta = {}
    for name in ["n337", "n537", "n726", "n926"]:
        text = (REF_NETS / f"{name}.net").read_text()
        fin, layers = parse_layers(text)
        npools = sum(1 for l in layers if l[0] != "conv")
        fov = ref.fov(text)
        ok = []
        for e in range(fov[0], fov[0] + 60):
            _, viol = ref.propagate(text, len(layers), npools, 1, (e, e, e), [1] * npools)
            if viol < 0:
                ok.append(e)
        shapes, viol = ref.propagate(text, len(layers), npools, 1, (ok[0],) * 3, [1] * npools)
        meta[name] = {"text": text, "fov": list(fov), "admissible_mpf": ok,
                      "chain_at_first": shapes.tolist()}
    (GOLD / "shapes.json").write_text(json.dumps(meta, indent=1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nets", action="store_true", help="also run the bundled nets (slow)")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    GOLD.mkdir(parents=True, exist_ok=True)
    ref = Ref(workers=0)
    steps = {"basic": gen_basic, "pools": gen_pools, "fft": gen_fft, "conv": gen_conv,
             "shapes": gen_shapes, "nets": lambda r: gen_nets(r, False)}
    if args.nets:
        steps = {"bundled": lambda r: gen_nets(r, True)}
    for name, fn in steps.items():
        if args.only and name not in args.only.split(","):
            continue
        t0 = time.time()
        fn(ref)
        print(f"golden {name}: {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
