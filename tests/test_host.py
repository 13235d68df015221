"""CPU: the C-ABI library loads, exports every symbol include/vxg.h declares,
and its host logic (grammar, shape rules, generators, padded sizes) matches
the reference's golden vectors.  No GPU compute is called here."""
import ctypes as C
import json
import re

import numpy as np
import pytest

from conftest import GOLD, ROOT


def declared_symbols():
    text = (ROOT / "include" / "vxg.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vxg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1606_05688_b200._lib import LIB_PATH
    lib = C.CDLL(str(LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_optimal_fft_size_matches_reference(golden):
    import paper_1606_05688_b200 as v
    g = golden("basic")
    for prof, key in [("host", "fft_size_host"), ("device", "fft_size_dev"), ("any", "fft_size_any")]:
        got = np.array([v.optimal_fft_size(int(n), prof) for n in g["fft_size_n"]])
        assert np.array_equal(got, g[key]), key
    with pytest.raises(ValueError):
        v.optimal_fft_size(0)


def test_generators_bit_exact(golden):
    import paper_1606_05688_b200 as v
    from oracle.make_golden import TOY_NETS
    g = golden("basic")
    assert np.array_equal(v.fill_random(4096, 7), g["fill_random_seed7_f32"])
    for name, text in TOY_NETS.items():
        net = v.parse_network_spec(text)
        assert np.array_equal(v.random_weights(net, 11), g[f"weights_{name}_seed11"]), name


def test_bundled_nets_fov_and_shapes():
    import paper_1606_05688_b200 as v
    from paper_1606_05688_b200.bundled_nets import FOV, NETS
    meta = json.loads((GOLD / "shapes.json").read_text())
    for name, text in NETS.items():
        net = v.parse_network_spec(text)
        ref = v.parse_network_spec(meta[name]["text"])  # the reference file, comments included
        assert net.format() == ref.format()
        assert net.field_of_view() == tuple(meta[name]["fov"]) == (FOV[name],) * 3
        fov = FOV[name]
        ok = [e for e in range(fov, fov + 60) if net.propagate(1, e)[1] < 0]
        assert ok == meta[name]["admissible_mpf"], name
        shapes, viol = net.propagate(1, ok[0])
        assert viol < 0
        assert [list(s) for s in shapes] == meta[name]["chain_at_first"]


def test_grammar_and_parse_errors():
    import paper_1606_05688_b200 as v
    net = v.parse_network_spec("# c\ninput 2\nconv 4 3 2 1 relu\npool 2 mpf\npool 1 2 3 plain\n"
                               "pool 2 auto\nconv 1 1\n")
    assert net.layers[0] == ("conv", 4, (3, 2, 1), True)
    assert net.layers[1] == ("pool", (2, 2, 2), "mpf")
    assert net.layers[2] == ("pool", (1, 2, 3), "plain")
    assert net.layers[3] == ("pool", (2, 2, 2), "auto")
    # round trip (netspec.hpp:101-103)
    assert v.parse_network_spec(net.format()).format() == net.format()
    bad = {
        "conv 1 1\n": (1, "missing input declaration"),
        "input 1\ninput 1\nconv 1 1\n": (2, "duplicate input declaration"),
        "input 1\nconv x 1\n": (2, "expected a number, got 'x'"),
        "input 1\nconv 1 0\n": (2, "extent must be >= 1"),
        "input 1\nfoo\n": (2, "unknown keyword 'foo'"),
        "input 1\npool 2 2\n": (2, "pool takes one or three window extents"),
        "input 1\n": (1, "network needs at least one layer"),
        "input 0\nconv 1 1\n": (1, "feature count must be >= 1"),
    }
    for text, (line, msg) in bad.items():
        with pytest.raises(v.ParseError) as ei:
            v.parse_network_spec(text)
        assert ei.value.line == line, text
        assert msg in str(ei.value), text


def test_propagate_rules():
    import paper_1606_05688_b200 as v
    net = v.parse_network_spec("input 1\nconv 2 3\npool 2\nconv 1 2\n")
    # MPF: (n+1) % p == 0 after the conv; plain: n % p == 0 (planner.cpp:563-583)
    shapes, viol = net.propagate(1, 9, [1])
    assert viol < 0 and shapes[2] == (8, 2, 3, 3, 3) and shapes[3] == (8, 1, 2, 2, 2)
    shapes, viol = net.propagate(1, 9, [0])
    assert viol == 1
    shapes, viol = net.propagate(1, 8, [0])
    assert viol < 0 and shapes[2] == (1, 2, 3, 3, 3)
    _, viol = net.propagate(1, 2, [1])
    assert viol == 0  # kernel larger than image
    with pytest.raises(ValueError):
        v.propagate_shapes(net, (1, 3, 8, 8, 8))


def test_library_refuses_without_gpu_cleanly():
    """Context creation without a CUDA device reports a status, never crashes."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1606_05688_b200 as v
    with pytest.raises((RuntimeError, ValueError)):
        v.Context(0)
