"""GPU parity of the device-resident network forward (execute_plan with an
all-fragment plan) against the reference run in fp64 on identical inputs and
weights (oracle/make_golden.py), for toy nets and all four bundled nets at
their smallest admissible extents; plus execution-shape invariants."""
import json

import numpy as np
import pytest

from conftest import GOLD, rel_error

pytestmark = pytest.mark.gpu

TOL = 1e-4  # north star: max-rel <= 1e-4 normalised by output magnitude


def _run(v, ctx, text, m, algos):
    net = v.parse_network_spec(text)
    w = v.random_weights(net, m["wseed"])
    x = v.fill_random(net.features_in * int(np.prod(m["extent"])), m["iseed"]).reshape(
        (1, net.features_in) + tuple(m["extent"]))
    out, rep = v.execute(net, w, x, ctx, conv_algos=algos)
    return out, rep


@pytest.mark.parametrize("algos", ["direct", "fft", None])
def test_toy_nets(golden, ctx, algos):
    import paper_1606_05688_b200 as v
    meta = json.loads((GOLD / "nets.json").read_text())
    g = golden("nets")
    for name, m in meta.items():
        out, rep = _run(v, ctx, m["text"], m, algos)
        assert out.shape == tuple(m["out_shape"])
        assert rel_error(out, g[f"{name}_out64"]) <= TOL, name
        assert rep.voxels == np.prod(m["out_shape"][2:])


@pytest.mark.parametrize("name", ["n337", "n726", "n926", "n537"])
def test_bundled_nets(golden, ctx, name):
    import paper_1606_05688_b200 as v
    meta = json.loads((GOLD / "nets_bundled.json").read_text())
    g = golden("nets_bundled")
    m = meta[name]
    out, rep = _run(v, ctx, m["text"], m, None)
    assert out.shape == tuple(m["out_shape"])
    err = rel_error(out, g[f"{name}_out64"])
    assert err <= TOL, err
    assert rep.seconds > 0 and len(rep.layer_seconds) == v.parse_network_spec(m["text"]).layer_count


@pytest.mark.parametrize("name", ["n537", "n726"])
def test_measured_planner_keeps_parity(golden, ctx, name):
    """The measured-time planner (Model.tune) only changes tile sizes and FFT vs
    direct: the bundled net still matches the fp64 reference, every conv layer
    reports a measured choice and a positive time estimate."""
    import paper_1606_05688_b200 as v
    meta = json.loads((GOLD / "nets_bundled.json").read_text())
    g = golden("nets_bundled")
    m = meta[name]
    net = v.parse_network_spec(m["text"])
    w = v.random_weights(net, m["wseed"])
    e = tuple(m["extent"])
    x = v.fill_random(int(np.prod(e)), m["iseed"]).reshape((1, 1) + e)
    model = v.Model(net, w, ctx)
    model.tune(1, e)
    plan = model.plan_info(1, e)
    convs = [l for l in plan if l["kind"] == "conv"]
    assert convs and all(l["seconds"] > 0 for l in plan)
    assert all(l["measured"] for l in convs if l["algo"] == "fft")
    for algos in (None, ["direct"] + ["auto"] * (len(convs) - 1)):
        out, rep = model.forward(x, conv_algos=algos)
        assert rel_error(out, g[f"{name}_out64"]) <= TOL, algos
    model.close()


def test_forward_many_matches_single_forwards(ctx):
    """The streaming API (double-buffered uploads / downloads on copy streams)
    returns, patch for patch, exactly what single forwards return."""
    import torch
    import paper_1606_05688_b200 as v
    from paper_1606_05688_b200.bundled_nets import NETS
    net = v.parse_network_spec(NETS["n337"])
    w = v.random_weights(net, 5)
    model = v.Model(net, w, ctx)
    xs = [torch.from_numpy(v.fill_random((1, 1, 100, 100, 100), 20 + i)).pin_memory().numpy() for i in range(3)]
    outs, sec = model.forward_many(xs)
    assert sec > 0 and len(outs) == 3
    for x, y in zip(xs, outs):
        want, _ = model.forward(x)
        assert np.array_equal(y, want)
    model.close()


def test_forward_independent_of_budget_and_algorithm(ctx):
    """Any feasible execution gives the same dense result (execute.hpp:384-386):
    fragment groups forced small by the budget reproduce the unconstrained run
    bit for bit (execute_test.cpp:188-227); FFT vs direct agree to tolerance."""
    import torch
    import paper_1606_05688_b200 as v
    from paper_1606_05688_b200.bundled_nets import NETS
    net = v.parse_network_spec(NETS["n337"])
    w = v.random_weights(net, 3)
    x = torch.from_numpy(v.fill_random((1, 1, 100, 100, 100), 9)).cuda()
    big, _ = v.Model(net, w, ctx).forward(x, conv_algos="fft")
    need = v.Model(net, w, ctx).plan_bytes(1, 100, "fft")
    assert need > 0
    tight = v.Context(0, budget_bytes=int(need * 1.3) + (64 << 20))
    small, _ = v.Model(net, w, tight).forward(x, conv_algos="fft")
    assert torch.equal(big, small)
    direct, _ = v.Model(net, w, ctx).forward(x, conv_algos="direct")
    err = ((direct - big).abs().max() / direct.abs().max()).item()
    assert err <= TOL
    tight.close()


def test_forward_translation_equivariance(ctx):
    """Dense out[d] depends only on in[d, d+fov): a crop at an offset gives the
    matching block of the full output (the large-config parity recipe)."""
    import torch
    import paper_1606_05688_b200 as v
    from paper_1606_05688_b200.bundled_nets import NETS
    net = v.parse_network_spec(NETS["n337"])
    w = v.random_weights(net, 1)
    model = v.Model(net, w, ctx)
    x = torch.from_numpy(v.fill_random((1, 1, 148, 148, 148), 1)).cuda()
    full, _ = model.forward(x)
    o = (24, 8, 40)
    crop = x[:, :, o[0]:o[0] + 100, o[1]:o[1] + 100, o[2]:o[2] + 100].contiguous()
    part, _ = model.forward(crop)
    ref = full[:, :, o[0]:o[0] + 16, o[1]:o[1] + 16, o[2]:o[2] + 16]
    err = ((part - ref).abs().max() / ref.abs().max()).item()
    assert err <= TOL, err


def test_forward_errors(ctx):
    import paper_1606_05688_b200 as v
    from paper_1606_05688_b200.bundled_nets import NETS
    net = v.parse_network_spec(NETS["n337"])
    w = v.random_weights(net, 1)
    with pytest.raises(ValueError, match="propagate"):
        v.execute(net, w, np.zeros((1, 1, 93, 93, 93), np.float32), ctx)
    tiny = v.Context(0, budget_bytes=64 << 20)
    with pytest.raises(v.ResourceExhausted):
        v.execute(net, w, np.zeros((1, 1, 148, 148, 148), np.float32), tiny)
    tiny.close()


def test_cpp_dropin_runs_bundled_net_unchanged(golden, tmp_path):
    """A reference-style C++ caller (include/voxin/*.hpp, the reference's API at
    T = float) runs the bundled n337 description through parse_network_spec ->
    random_weights<float> -> optimize_plan -> execute_plan."""
    import subprocess
    from conftest import ROOT
    meta = json.loads((GOLD / "nets_bundled.json").read_text())["n337"]
    exe = tmp_path / "shim_net"
    lib = ROOT / "paper_1606_05688_b200"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "shim_net.cpp"), "-L", str(lib), "-lvxg",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    net_file = tmp_path / "n337.net"
    net_file.write_text(meta["text"])
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), str(net_file), str(meta["extent"][0]), str(meta["wseed"]),
                        str(meta["iseed"]), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
    got = np.fromfile(out, np.float32).reshape(meta["out_shape"])
    assert rel_error(got, golden("nets_bundled")["n337_out64"]) <= TOL


def test_tiled_volume_equals_whole_volume(ctx):
    """Halo tiles (the multi-GPU sharding unit) stitch to the whole-volume output."""
    import paper_1606_05688_b200 as v
    from paper_1606_05688_b200 import tiler
    from paper_1606_05688_b200.bundled_nets import NETS
    net = v.parse_network_spec(NETS["n337"])
    model = v.Model(net, v.random_weights(net, 5), ctx)
    vol = v.fill_random((1, 1, 140, 132, 124), 17)
    dense = tiler.infer_volume(model, vol, (24, 24, 16))
    # reference: each 8-aligned output block from one big forward of the largest admissible crop
    full, _ = model.forward(np.ascontiguousarray(vol[:, :, :132, :132, :124]))
    assert dense.shape == (1, 3, 56, 48, 40)
    err = np.abs(dense[:, :, :48, :48, :40] - full).max() / np.abs(full).max()
    assert err <= TOL, err


def _bench_plan(name, ctx):
    """The bench's model, patch and plan for a bundled net (bench.choose_patch
    after vxg_model_tune), weights random_weights(net, 1) as the bench uses."""
    import importlib.util
    import paper_1606_05688_b200 as v
    from paper_1606_05688_b200.bundled_nets import FOV, NETS
    from conftest import ROOT
    spec = importlib.util.spec_from_file_location("_bench", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    net = v.parse_network_spec(NETS[name])
    fov = FOV[name]
    model = v.Model(net, v.random_weights(net, 1), ctx)
    # the context's budget was fixed when the session's context was made; tensors
    # torch still caches from earlier tests are outside it, so also cap by what
    # the device has free now (bench.py runs in a fresh process: budget only)
    import gc
    import torch
    gc.collect()
    torch.cuda.empty_cache()
    ctx.trim()
    budget = min(ctx.memory()["budget"] - ctx.memory()["current"],
                 torch.cuda.mem_get_info()[0] - (3 << 30))
    e, _ = bench.choose_patch(model, net, fov, budget, False)
    model.tune(1, e)
    e, algos = bench.choose_patch(model, net, fov, budget, True)
    return v, net, fov, model, e, algos


# smallest admissible patch of each bundled net: the reference
# CPU path finishes one forward there in ~20-60 s on the GPU box's host cores
REF_CROP = {"n537": 170, "n726": 120, "n926": 158}


@pytest.mark.parametrize("name,blocks", [("n537", 2), ("n726", 1), ("n926", 1)])
def test_bench_patch_vs_reference_crops(ctx, name, blocks):
    """Headline-config parity against the REFERENCE itself (SURVEY 8c recipe):
    the bundled net at the bench's own patch (largest fitting the HBM budget)
    with the bench's own plan (measured planner: direct tensor-core first layer
    fused with its MPF, tcgen05 FFT layers), and at random offsets o the dense
    block out[o : o + c - fov + 1] against the reference library (oracle/_ref,
    unmodified sources, fp32 execute_plan with fft_task_parallel convs and MPF
    pools) run on the matching c^3 input crop -- translation equivariance makes
    the crop an exact sub-problem.  Tolerance: the north star's 1e-4 max-rel."""
    import torch
    from oracle.refbind import REF_SO, Ref
    from paper_1606_05688_b200.bundled_nets import NETS
    assert REF_SO.exists(), "oracle/_ref/libvoxref.so missing (built by __graft_entry__.build())"
    v, net, fov, model, e, algos = _bench_plan(name, ctx)
    c = REF_CROP[name]
    x_host = v.fill_random((1, 1, e, e, e), 11)
    full, _ = model.forward(torch.from_numpy(x_host).cuda(), conv_algos=algos)
    assert tuple(full.shape) == (1, net.features_out) + (e - fov + 1,) * 3
    ref = Ref(workers=0)
    rng = np.random.default_rng(7)
    n = c - fov + 1
    for b in range(blocks):
        o = [int(t) for t in rng.integers(0, e - c + 1, size=3)] if b == 0 else [e - c] * 3
        crop = np.ascontiguousarray(x_host[:, :, o[0]:o[0] + c, o[1]:o[1] + c, o[2]:o[2] + c])
        want, _ = ref.net_forward(NETS[name], 1, crop, conv_kind=3, prec=32,
                                  out_shape=(1, net.features_out, n, n, n))
        got = full[:, :, o[0]:o[0] + n, o[1]:o[1] + n, o[2]:o[2] + n].cpu().numpy()
        err = rel_error(got, want)
        print(f"{name} patch {e}^3 plan {algos}: block at {o} rel err {err:.2e}")
        assert err <= TOL, (name, e, o, err)
    del full
    model.close()
    torch.cuda.empty_cache()


def test_bench_patch_full_size_vs_direct_crops(ctx):
    """BASELINE-size cross-check on the GPU, wider than the reference blocks
    above: n537 on the bench's patch with the bench's plan, at three random 16^3
    output blocks against all-direct forwards of the matching input crops.  The
    FFT layers (tcgen05 3xTF32 contraction, tile transforms) are checked against
    the FFMA direct convolution; the first conv + MPF pair runs the same
    tensor-core direct kernel with the same slab-fused MPF in both forwards (f = 1,
    80 maps), so it is pinned by the reference-crop test above, not here."""
    import torch
    v, net, fov, model, e, algos = _bench_plan("n537", ctx)
    c = 186
    plan = model.plan_info(1, e, algos)
    assert any(l.get("tc") for l in plan if l["kind"] == "conv"), plan
    x = torch.from_numpy(v.fill_random((1, 1, e, e, e), 11)).cuda()
    full, _ = model.forward(x, conv_algos=algos)
    assert tuple(full.shape) == (1, 3, e - fov + 1, e - fov + 1, e - fov + 1)
    rng = np.random.default_rng(3)
    for _ in range(3):
        o = [int(t) for t in rng.integers(0, e - c + 1, size=3)]
        crop = x[:, :, o[0]:o[0] + c, o[1]:o[1] + c, o[2]:o[2] + c].contiguous()
        part, _ = model.forward(crop, conv_algos="direct")
        n = c - fov + 1
        ref = full[:, :, o[0]:o[0] + n, o[1]:o[1] + n, o[2]:o[2] + n]
        err = ((part - ref).abs().max() / part.abs().max()).item()
        assert err <= TOL, (o, err)
    del full
    model.close()
    torch.cuda.empty_cache()


def test_network_forward_rejects_nan_input(ctx):
    """mpf_pool's check_no_nan (layers.hpp:111-116, :429) inside the network
    forward: a NaN voxel reaches the first MPF through an identity first conv ->
    std::invalid_argument / ValueError, for host and device inputs; the flag
    does not leak into the next (clean) forward.  (After a ReLU conv the NaN is
    gone, in the reference as here: activate() maps NaN to 0, layers.hpp:105-108.)"""
    import torch
    import paper_1606_05688_b200 as v
    net = v.parse_network_spec("input 1\nconv 4 3\npool 2 mpf\nconv 4 3 relu\npool 2 mpf\nconv 2 3\n")
    w = v.random_weights(net, 9003)
    model = v.Model(net, w, ctx)
    x = v.fill_random((1, 1, 21, 21, 21), 9103)
    bad = x.copy()
    bad[0, 0, 10, 11, 12] = np.nan
    for algos in ("direct", "fft"):
        with pytest.raises(ValueError, match="NaN"):
            model.forward(bad, conv_algos=algos)
        with pytest.raises(ValueError, match="NaN"):
            model.forward(torch.from_numpy(bad).cuda(), conv_algos=algos)
        out, _ = model.forward(x, conv_algos=algos)
        assert np.isfinite(out).all()
    with pytest.raises(ValueError, match="NaN"):
        model.forward_many([bad, x])
    # a network starting with a pool rejects a NaN input directly
    pnet = v.parse_network_spec("input 1\npool 2 mpf\nconv 2 3\n")
    pm = v.Model(pnet, v.random_weights(pnet, 1), ctx)
    with pytest.raises(ValueError, match="NaN"):
        pm.forward(bad)


def test_run_bench_csv_matches_the_reference_columns(tmp_path):
    """tools/run_bench.py (the device `voxinfer bench`, proj/src/cli.cpp:225-280):
    header and one row per admissible extent, memory columns in scalars, layer
    times summing to the forward.  memory_model is the plan's minimum-footprint
    schedule; the forward grows its fragment groups into the free budget, so its
    audited peak lies between half that and the context budget."""
    import csv
    import importlib.util
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    spec = importlib.util.spec_from_file_location("run_bench", root / "tools" / "run_bench.py")
    rb = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(rb)
    import gc
    import torch
    import paper_1606_05688_b200 as v
    gc.collect()
    torch.cuda.empty_cache()  # tensors earlier tests left in torch's cache
    budget = v.default_context().memory()["budget"]
    out = tmp_path / "bench.csv"
    assert rb.main(["--net", "n337", "--min-extent", "92", "--max-extent", "108", "--csv", str(out)]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0][:5] == ["input_extent", "memory_model", "memory_audited", "voxels_per_sec", "seconds"]
    assert rows[0][5:] == [f"layer{i}_ms" for i in range(len(rows[0]) - 5)]
    assert len(rows) >= 3
    for r in rows[1:]:
        e, model, audited, vps, sec = int(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4])
        assert vps > 0 and sec > 0 and model > 0 and 0.5 * model <= audited <= budget / 4
        assert abs(sum(float(x) for x in r[5:]) * 1e-3 - sec) <= 0.25 * sec


def test_held_arena_yields_to_other_contexts():
    """The forward's arena block stays with its context between forwards (no
    pool remap per forward) but is not charged while idle, and yields to a new
    context's budget and to Context.trim() (vxg_ctx_trim)."""
    import torch
    import paper_1606_05688_b200 as v
    from paper_1606_05688_b200.bundled_nets import NETS
    net = v.parse_network_spec(NETS["n337"])
    a = v.Context(0)
    m = v.Model(net, v.random_weights(net, 1), a)
    x = torch.from_numpy(v.fill_random((1, 1, 148, 148, 148), 3)).cuda()
    y1, _ = m.forward(x)
    assert a.memory()["current"] < 4 * 2 ** 30  # weights and spectra only: the idle block is not charged
    y2, _ = m.forward(x)                         # reuses the held block
    assert torch.equal(y1, y2)
    b = v.Context(0)                             # creation hands idle caches back first
    assert b.memory()["budget"] > 100 * 2 ** 30
    a.trim()
    y3, _ = m.forward(x)
    assert torch.equal(y1, y3)
    m.close()
