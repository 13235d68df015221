"""CPU: pin the plain-C oracle (oracle/voxin_oracle.c) against golden vectors
produced by the UNMODIFIED reference (oracle/make_golden.py).  Once these pass,
the oracle is a trustworthy checker for the GPU parity tests."""
import json

import numpy as np
import pytest

from conftest import GOLD, rel_error


def test_generators_bit_exact(golden, oracle):
    g = golden("basic")
    assert np.array_equal(oracle.fill_random(4096, 7), g["fill_random_seed7_f32"])
    from oracle.make_golden import TOY_NETS, parse_layers
    for name, text in TOY_NETS.items():
        fin, layers = parse_layers(text)
        convs, f = [], fin
        for l in layers:
            if l[0] == "conv":
                convs.append((l[1], f, int(np.prod(l[2]))))
                f = l[1]
        assert np.array_equal(oracle.random_weights(convs, 11), g[f"weights_{name}_seed11"]), name


def test_optimal_fft_size(golden, oracle):
    g = golden("basic")
    for prof, key in [(0, "fft_size_host"), (1, "fft_size_dev"), (2, "fft_size_any")]:
        got = [oracle.optimal_fft_size(int(n), prof) for n in g["fft_size_n"]]
        assert np.array_equal(np.array(got), g[key]), key
    # fft_test.cpp:17-24 pinned values
    assert oracle.optimal_fft_size(121, 0) == 125
    assert oracle.optimal_fft_size(11, 1) == 12
    assert oracle.optimal_fft_size(143, 0) == 144
    assert oracle.optimal_fft_size(143, 2) == 143


def test_pools_and_recombine(golden, oracle):
    g = golden("pools")
    assert np.array_equal(oracle.pool(False, g["pin_pool_in"], (1, 1, 2)), g["pin_pool_out"])
    assert np.array_equal(oracle.pool(True, g["pin_mpf_in"], (1, 1, 2)), g["pin_mpf_out"])
    assert g["pin_mpf_out"].reshape(-1).tolist() == [5, 3, 5, 9]  # layers_test.cpp:72-82
    for i in range(int(g["ncases"])):
        got = oracle.pool(bool(g[f"case{i}_kind"]), g[f"case{i}_in"], tuple(g[f"case{i}_p"]))
        assert np.array_equal(got, g[f"case{i}_out"]), i
    assert np.array_equal(oracle.recombine(g["pin_rec_in"], [(1, 1, 2)], 1), g["pin_rec_out"])
    assert g["pin_rec_out"].reshape(-1).tolist() == [1, 3, 2, 4]  # layers_test.cpp:113-124
    for i in range(int(g["nrec"])):
        wins = [tuple(w) for w in g[f"rec{i}_win"]]
        got = oracle.recombine(g[f"rec{i}_in"], wins, int(g[f"rec{i}_S0"]))
        assert np.array_equal(got, g[f"rec{i}_out"]), i


def test_transforms(golden, oracle):
    g = golden("fft")
    for i in range(int(g["ncases"])):
        pad = tuple(g[f"p{i}_pad"])
        n = tuple(g[f"p{i}_n"])
        if np.prod(pad) > 4000:
            continue  # the O(N^2)-per-line DFT oracle: small cases only
        assert rel_error(oracle.pruned_fwd(g[f"p{i}_in"], pad), g[f"p{i}_nested"]) < 1e-12
        assert rel_error(oracle.pruned_inv(g[f"p{i}_nested"], pad, n), g[f"p{i}_inv"]) < 1e-12
        assert rel_error(oracle.batched_fwd(g[f"p{i}_bin"], pad), g[f"p{i}_batched"]) < 1e-12
        assert rel_error(oracle.batched_inv(g[f"p{i}_batched"], pad, n), g[f"p{i}_binv"]) < 1e-12


def test_conv(golden, oracle):
    g = golden("conv")
    for i in range(int(g["ncases"])):
        x, w, b = g[f"c{i}_in"], g[f"c{i}_w"], g[f"c{i}_b"]
        if x.shape[1] * w.shape[0] > 1000:
            continue  # 80x80 case: covered on the GPU against the golden output
        got = oracle.conv(x, w, b, bool(g[f"c{i}_relu"]))
        assert rel_error(got, g[f"c{i}_out64"]) < 1e-12, i
        # the reference's own fp32 FFT path agrees with its fp64 direct path
        assert rel_error(g[f"c{i}_fft32"], g[f"c{i}_out64"]) < 1e-5, i


def test_toy_nets(golden, oracle):
    meta = json.loads((GOLD / "nets.json").read_text())
    g = golden("nets")
    from oracle.make_golden import parse_layers
    for name, m in meta.items():
        fin, layers = parse_layers(m["text"])
        convs, f = [], fin
        for l in layers:
            if l[0] == "conv":
                convs.append((l[1], f, int(np.prod(l[2]))))
                f = l[1]
        w = oracle.random_weights(convs, m["wseed"])
        x = oracle.fill_random(fin * int(np.prod(m["extent"])), m["iseed"]).reshape(
            (1, fin) + tuple(m["extent"]))
        got = oracle.net_forward(layers, w, x)
        assert got.shape == tuple(m["out_shape"])
        assert rel_error(got, g[f"{name}_out64"]) < 1e-6, name


def test_reference_stepper_is_execute_plan():
    """bench.py's reference arm runs execute_plan's host-only path one layer per
    step (oracle/ref_shim.cpp ref_stepper_*): a completed stepped forward equals
    the reference's execute_plan on the same plan bit for bit, forward after
    forward, and the planner variant takes the reference planner's own kinds."""
    from oracle.refbind import REF_SO, Ref
    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built")
    ref = Ref(2)
    net = "input 1\nconv 4 3 relu\npool 2 mpf\nconv 4 3 relu\npool 2 mpf\nconv 2 3\n"
    x = ref.fill_random(21 ** 3, 5).reshape(1, 1, 21, 21, 21)
    st = ref.stepper(net, 21, 1, 5, plan="forced", conv_kind=3)
    assert st.kinds == ["fft-task-parallel", "pool-fragments"] * 2 + ["fft-task-parallel"]
    for _ in range(2):
        steps = [st.step() for _ in range(5)]
        assert [s[0] for s in steps] == list(range(5)) and steps[-1][2]
        got = st.output()
        want, _ = ref.net_forward(net, 1, x, conv_kind=3, prec=32, out_shape=got.shape)
        assert got.tobytes() == want.tobytes()
    pl = ref.stepper(net, 21, 1, 5, plan="planner")
    assert len(pl.kinds) == 5 and pl.kinds[1] in ("pool-fragments", "pool-plain")
