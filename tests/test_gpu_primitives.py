"""GPU parity of every layer primitive and transform against the reference's
golden vectors (oracle/make_golden.py) and the C oracle, through the C-ABI.

Tolerances (north star: fp32, max-rel <= 1e-4 normalised by output magnitude):
  * pools, MPF fragment order, recombination: bit-exact;
  * convolutions: rel_error <= 1e-5 (direct) / 1e-4 (tiled FFT) vs fp64 reference;
  * transforms: rel_error <= 1e-5 vs fp64 reference.
"""
import numpy as np
import pytest

from conftest import rel_error

pytestmark = pytest.mark.gpu


def _cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_pools_bit_exact(golden, ctx):
    import paper_1606_05688_b200 as v
    g = golden("pools")
    out = v.max_pool(g["pin_pool_in"], (1, 1, 2), ctx).output
    assert np.array_equal(out, g["pin_pool_out"])
    out = v.mpf_pool(g["pin_mpf_in"], (1, 1, 2), ctx).output
    assert out.reshape(-1).tolist() == [5, 3, 5, 9]
    for i in range(int(g["ncases"])):
        fn = v.mpf_pool if int(g[f"case{i}_kind"]) else v.max_pool
        p = tuple(int(x) for x in g[f"case{i}_p"])
        host = fn(g[f"case{i}_in"], p, ctx).output
        assert np.array_equal(host, g[f"case{i}_out"]), i
        dev = fn(_cuda(g[f"case{i}_in"]), p, ctx).output
        assert np.array_equal(dev.cpu().numpy(), g[f"case{i}_out"]), i


def test_mpf_random_vs_oracle_and_signed_zero(oracle, ctx):
    import paper_1606_05688_b200 as v
    rng = np.random.default_rng(5)
    for shape, p in [((2, 3, 11, 9, 7), (2, 2, 2)), ((1, 2, 8, 11, 5), (3, 2, 3)),
                     ((3, 1, 1, 1, 9), (1, 1, 5))]:
        x = rng.standard_normal(shape).astype(np.float32)
        x[x > 1.0] = 0.0
        x[x < -1.0] = -0.0  # ties between +0 / -0 must resolve like the reference scan
        got = v.mpf_pool(x, p, ctx).output
        want = oracle.pool(True, x, p)
        assert got.tobytes() == want.tobytes()


def test_pool_errors(ctx):
    import paper_1606_05688_b200 as v
    with pytest.raises(ValueError, match="divisible"):
        v.max_pool(np.zeros((1, 1, 5, 4, 4), np.float32), (2, 2, 2), ctx)
    with pytest.raises(ValueError, match="extent\\+1"):
        v.mpf_pool(np.zeros((1, 1, 4, 5, 5), np.float32), (2, 2, 2), ctx)
    x = np.zeros((1, 1, 2, 2, 2), np.float32)
    x.reshape(-1)[3] = np.nan
    with pytest.raises(ValueError, match="NaN"):
        v.max_pool(x, (1, 1, 1), ctx)
    with pytest.raises(ValueError, match="NaN"):
        v.mpf_pool(np.full((1, 1, 3, 3, 3), np.nan, np.float32), (2, 2, 2), ctx)
    # window 1 is the identity (layers_test.cpp:106-108)
    y = np.random.default_rng(1).standard_normal((2, 2, 3, 4, 5)).astype(np.float32)
    assert np.array_equal(v.mpf_pool(y, (1, 1, 1), ctx).output, y)


def test_recombine_bit_exact(golden, ctx):
    import paper_1606_05688_b200 as v
    g = golden("pools")
    assert v.recombine_fragments(g["pin_rec_in"], [(1, 1, 2)], 1, ctx).reshape(-1).tolist() == [1, 3, 2, 4]
    for i in range(int(g["nrec"])):
        wins = [tuple(int(x) for x in w) for w in g[f"rec{i}_win"]]
        got = v.recombine_fragments(g[f"rec{i}_in"], wins, int(g[f"rec{i}_S0"]), ctx)
        assert np.array_equal(got, g[f"rec{i}_out"]), i
        got = v.recombine_fragments(_cuda(g[f"rec{i}_in"]), wins, int(g[f"rec{i}_S0"]), ctx)
        assert np.array_equal(got.cpu().numpy(), g[f"rec{i}_out"]), i
    t = np.random.default_rng(3).standard_normal((3, 2, 2, 3, 4)).astype(np.float32)
    assert np.array_equal(v.recombine_fragments(t, [], 3, ctx), t)
    with pytest.raises(ValueError, match="mismatch"):
        v.recombine_fragments(t, [(2, 2, 2)], 3, ctx)


@pytest.mark.parametrize("wins,n", [([(2, 2, 2), (2, 2, 2)], (151, 150, 149)),
                                    ([(2, 2, 2)] * 3, (75, 74, 76)),
                                    ([(3, 2, 1), (1, 2, 3)], (60, 61, 62))])
def test_recombine_large_vs_numpy(ctx, wins, n):
    """Large fragment tensors (the bench's recombine sizes) against a numpy
    restatement of recombine_fragments (layers.hpp:477-520)."""
    import torch
    import paper_1606_05688_b200 as v
    alpha = int(np.prod([np.prod(w) for w in wins]))
    S0, f = 2, 3
    rng = np.random.default_rng(len(wins))
    frag = rng.standard_normal((S0 * alpha, f) + n).astype(np.float32)
    got = v.recombine_fragments(torch.from_numpy(frag).cuda(), wins, S0, ctx).cpu().numpy()
    stride = [int(np.prod([w[a] for w in wins])) for a in range(3)]
    want = np.empty((S0, f) + tuple(stride[a] * n[a] for a in range(3)), np.float32)
    # fragment index: first pool's offset slowest; offset along axis a adds o * (stride before pool)
    for s in range(S0):
        for b in range(alpha):
            rem, off = b, [0, 0, 0]
            for wi in range(len(wins)):
                vol = int(np.prod([np.prod(w) for w in wins[wi + 1:]])) if wi + 1 < len(wins) else 1
                idx, rem = divmod(rem, vol)
                w = wins[wi]
                o = (idx // (w[1] * w[2]), (idx // w[2]) % w[1], idx % w[2])
                pre = [int(np.prod([ww[a] for ww in wins[:wi]])) for a in range(3)]
                for a in range(3):
                    off[a] += o[a] * pre[a]
            want[s, :, off[0]::stride[0], off[1]::stride[1], off[2]::stride[2]] = frag[s * alpha + b]
    assert np.array_equal(got, want)


def test_mpf_then_recombine_is_dense_max_filter(ctx):
    """layers_test.cpp:134-158: MPF + recombination == dense max filter, exactly."""
    import paper_1606_05688_b200 as v
    x = np.random.default_rng(34).standard_normal((2, 2, 9, 7, 11)).astype(np.float32)
    p = (2, 2, 2)
    frag = v.mpf_pool(x, p, ctx).output
    dense = v.recombine_fragments(frag, [p], 2, ctx)
    want = np.full((2, 2, 8, 6, 10), -np.inf, np.float32)
    for qx in range(2):
        for qy in range(2):
            for qz in range(2):
                want = np.maximum(want, x[:, :, qx:qx + 8, qy:qy + 6, qz:qz + 10])
    assert np.array_equal(dense, want)


@pytest.mark.parametrize("algo", ["direct", "fft"])
def test_conv_matches_reference(golden, ctx, algo):
    import paper_1606_05688_b200 as v
    g = golden("conv")
    tol = 1e-5 if algo == "direct" else 1e-4
    fn = v.conv_direct if algo == "direct" else v.conv_fft_task_parallel
    for i in range(int(g["ncases"])):
        p = v.ConvLayerParams(g[f"c{i}_w"], g[f"c{i}_b"], "relu" if int(g[f"c{i}_relu"]) else "identity")
        res = fn(g[f"c{i}_in"], p, ctx)
        err = rel_error(res.output, g[f"c{i}_out64"])
        assert err <= tol, (i, err)
        assert res.audit.peak > 0


def test_conv_device_pointers_and_fft_variants(golden, ctx):
    import paper_1606_05688_b200 as v
    g = golden("conv")
    i = 6  # the 80 -> 80 k5 layer
    p = v.ConvLayerParams(_cuda(g[f"c{i}_w"]), _cuda(g[f"c{i}_b"]), "relu")
    for fn in (v.conv_fft_data_parallel, v.conv_fft_staged, v.conv_fft_task_parallel, v.conv_direct):
        out = fn(_cuda(g[f"c{i}_in"]), p, ctx).output
        assert rel_error(out.cpu().numpy(), g[f"c{i}_out64"]) <= 1e-4


@pytest.mark.parametrize("case", [
    (2, 8, (20, 18, 17), 8, (5, 3, 4)),
    (1, 1, (40, 33, 35), 16, (4, 4, 4)),
    (3, 4, (9, 9, 9), 5, (9, 9, 9)),
    (1, 6, (30, 30, 30), 3, (7, 7, 7)),
    (2, 5, (12, 13, 14), 7, (1, 1, 1)),
])
def test_conv_random_vs_oracle(oracle, ctx, case):
    import paper_1606_05688_b200 as v
    S, f, n, fo, k = case
    rng = np.random.default_rng(sum(n) + fo)
    x = rng.uniform(-1, 1, (S, f) + n).astype(np.float32)
    w = (rng.uniform(-1, 1, (fo, f) + k) * np.sqrt(3.0 / (f * np.prod(k)))).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
    want = oracle.conv(x, w, b, True)
    p = v.ConvLayerParams(w, b, "relu")
    assert rel_error(v.conv_direct(x, p, ctx).output, want) <= 1e-5
    assert rel_error(v.conv_fft_staged(x, p, ctx).output, want) <= 1e-4


@pytest.mark.parametrize("case", [
    (2, (30, 20, 300), 80, (2, 2, 2)),
    (1, (17, 19, 140), 48, (3, 3, 3)),
    (2, (24, 21, 131), 64, (4, 4, 4)),
    (1, (9, 10, 257), 80, (4, 3, 2)),
    (1, (9, 10, 40), 32, (4, 4, 4)),   # 32 maps: FFMA kernel
    # kz = 7 / 8 with nz % 4 != 0: the 16-byte superset of a staged row is up
    # to 3 floats longer than 128 + kz - 1 (row overflow)
    (1, (9, 10, 257), 48, (3, 3, 7)),
    (1, (8, 9, 259), 64, (2, 2, 8)),
    (1, (7, 8, 261), 80, (1, 2, 9)),
])
def test_conv_direct_single_input_map_tensor_cores(oracle, ctx, case):
    """f = 1 direct convolution (the first layer of every bundled net) on the
    tcgen05 implicit-GEMM kernel (48..80 maps per launch): several 128-voxel z
    tiles with a ragged last one, k^3 taps padded to 8/32/64, anisotropic
    kernels; against the C oracle (fp64)."""
    import paper_1606_05688_b200 as v
    S, n, fo, k = case
    rng = np.random.default_rng(sum(n) + fo)
    x = rng.uniform(-1, 1, (S, 1) + n).astype(np.float32)
    w = (rng.uniform(-1, 1, (fo, 1) + k) * np.sqrt(3.0 / np.prod(k))).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
    want = oracle.conv(x, w, b, True)
    got = v.conv_direct(x, v.ConvLayerParams(w, b, "relu"), ctx).output
    assert rel_error(got, want) <= 1e-5
    lin = v.conv_direct(x, v.ConvLayerParams(w, b, "identity"), ctx).output
    assert rel_error(lin, oracle.conv(x, w, b, False)) <= 1e-5


@pytest.mark.parametrize("variant", ["tc_pair", "tc_single", "ffma"])
def test_conv_fft_every_tile_size_vs_oracle(oracle, ctx, variant):
    """Every tile FFT size the planner may pick, each contraction and forward
    transform kernel, with several tiles per axis, ragged edges, an anisotropic
    kernel and a chunked spectrum (multi-launch) -- against the C oracle."""
    import paper_1606_05688_b200 as v
    S, f, fo = 2, 16, 16
    rng = np.random.default_rng(11)
    for T in v.TILE_SIZES:
        k = (min(3, T), min(2, T), min(3, T))
        n = (T + 7, 2 * T - 1, T + 3)
        x = rng.uniform(-1, 1, (S, f) + n).astype(np.float32)
        w = (rng.uniform(-1, 1, (fo, f) + k) * np.sqrt(3.0 / (f * np.prod(k)))).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
        want = oracle.conv(x, w, b, True)
        p = v.ConvLayerParams(w, b, "relu")
        got = v.conv_fft_tiled(x, p, T, tensor_cores=variant != "ffma", cta_pair=variant == "tc_pair",
                               spectra_budget=3 * (f + fo) * T * T * (T // 2 + 1) * 8 + 4096, ctx=ctx)
        assert rel_error(got, want) <= 1e-4, (T, variant, rel_error(got, want))


@pytest.mark.parametrize("fo", [32, 48, 64, 80])
def test_conv_fft_tensor_core_map_counts(oracle, ctx, fo):
    """Every output-map count the tcgen05 contraction instantiates (its TMEM
    accumulator split differs per count), several m-blocks and chunks."""
    import paper_1606_05688_b200 as v
    S, f, k, T = 3, 24, (3, 3, 3), 16
    n = (2 * (T - 2) + 2, 3 * (T - 2) + 2, T + 5)
    rng = np.random.default_rng(fo)
    x = rng.uniform(-1, 1, (S, f) + n).astype(np.float32)
    w = (rng.uniform(-1, 1, (fo, f) + k) * np.sqrt(3.0 / (f * 27))).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
    want = oracle.conv(x, w, b, True)
    p = v.ConvLayerParams(w, b, "relu")
    got = v.conv_fft_tiled(x, p, T, tensor_cores=True, ctx=ctx)
    assert rel_error(got, want) <= 1e-4, rel_error(got, want)


def test_conv_fft_pair_major_spectrum_path(oracle, ctx, monkeypatch):
    """The optional pair-major Y layout (VXG_YPAIR=1: transposing tcgen05
    epilogue + TMA-gathered CTA-pair inverse) against the C oracle."""
    import paper_1606_05688_b200 as v
    monkeypatch.setenv("VXG_YPAIR", "1")
    S, f, fo = 2, 16, 32
    rng = np.random.default_rng(5)
    for T in (24, 32):
        k = (3, 4, 5)
        n = (T + 9, 2 * T - 3, T + 4)
        x = rng.uniform(-1, 1, (S, f) + n).astype(np.float32)
        w = (rng.uniform(-1, 1, (fo, f) + k) * np.sqrt(3.0 / (f * 60))).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
        got = v.conv_fft_tiled(x, v.ConvLayerParams(w, b, "relu"), T, ctx=ctx)
        assert rel_error(got, oracle.conv(x, w, b, True)) <= 1e-4, T


def test_conv_fft_pair_kernel_matches_single(ctx):
    """The CTA-pair forward transform computes the same transform as the one-CTA
    kernel (T = 32, an 80 -> 80 layer: the bench's deep-layer shape).  The two
    pair z lines differently in their two-for-one real transforms, so they
    agree to fp32 rounding, not bitwise."""
    import torch
    import paper_1606_05688_b200 as v
    gen = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand((3, 80, 60, 61, 59), device="cuda", generator=gen) * 2 - 1
    w = (torch.rand((80, 80, 5, 5, 5), device="cuda", generator=gen) * 2 - 1) * (3.0 / (80 * 125)) ** 0.5
    b = (torch.rand((80,), device="cuda", generator=gen) * 2 - 1) * 0.1
    p = v.ConvLayerParams(w.contiguous(), b.contiguous(), "relu")
    a = v.conv_fft_tiled(x, p, 32, cta_pair=True, ctx=ctx)
    c = v.conv_fft_tiled(x, p, 32, cta_pair=False, ctx=ctx)
    d = v.conv_direct(x, p, ctx).output
    scale = d.abs().max().item()
    assert (a - c).abs().max().item() / scale <= 2e-6
    assert (a - d).abs().max().item() / scale <= 1e-4


def test_conv_fft_vs_direct_large(ctx):
    """Size-independent property at a realistic layer size: FFT == direct."""
    import torch
    import paper_1606_05688_b200 as v
    gen = torch.Generator(device="cuda").manual_seed(7)
    x = torch.rand((2, 80, 70, 70, 70), device="cuda", generator=gen) * 2 - 1
    w = (torch.rand((80, 80, 5, 5, 5), device="cuda", generator=gen) * 2 - 1) * (3.0 / (80 * 125)) ** 0.5
    b = (torch.rand((80,), device="cuda", generator=gen) * 2 - 1) * 0.1
    p = v.ConvLayerParams(w.contiguous(), b.contiguous(), "relu")
    a = v.conv_direct(x, p, ctx).output
    c = v.conv_fft_staged(x, p, ctx).output
    err = (a - c).abs().max().item() / a.abs().max().item()
    assert err <= 1e-4, err


def test_conv_errors(ctx):
    import paper_1606_05688_b200 as v
    x = np.zeros((1, 2, 4, 4, 4), np.float32)
    with pytest.raises(ValueError):
        v.conv_direct(x, v.ConvLayerParams(np.zeros((1, 3, 2, 2, 2), np.float32), np.zeros(1, np.float32)), ctx)
    with pytest.raises(ValueError):
        v.conv_direct(x, v.ConvLayerParams(np.zeros((1, 2, 5, 2, 2), np.float32), np.zeros(1, np.float32)), ctx)
    with pytest.raises(ValueError):
        v.conv_direct(x, v.ConvLayerParams(np.zeros((2, 2, 2, 2, 2), np.float32), np.zeros(1, np.float32)), ctx)


def test_conv_budget_exhausted():
    import paper_1606_05688_b200 as v
    small = v.Context(0, budget_bytes=1 << 20)
    x = np.zeros((1, 8, 40, 40, 40), np.float32)  # 2 MB input alone
    p = v.ConvLayerParams(np.zeros((8, 8, 3, 3, 3), np.float32), np.zeros(8, np.float32))
    with pytest.raises(v.ResourceExhausted):
        v.conv_fft_staged(x, p, small)
    assert small.memory()["current"] == 0  # every charge unwound (layers_test.cpp:416-432)
    small.close()


def test_transforms_match_reference(golden, ctx):
    import paper_1606_05688_b200 as v
    g = golden("fft")
    for i in range(int(g["ncases"])):
        pad = tuple(int(x) for x in g[f"p{i}_pad"])
        n = tuple(int(x) for x in g[f"p{i}_n"])
        assert rel_error(v.pruned_fft_forward(g[f"p{i}_in"], pad, ctx), g[f"p{i}_nested"]) <= 1e-5
        assert rel_error(v.pruned_fft_inverse(g[f"p{i}_nested"].astype(np.complex64), pad, n, ctx),
                         g[f"p{i}_inv"]) <= 1e-5
        assert rel_error(v.batched_fft_forward(g[f"p{i}_bin"], pad, ctx), g[f"p{i}_batched"]) <= 1e-5
        assert rel_error(v.batched_fft_inverse(g[f"p{i}_batched"].astype(np.complex64), pad, n, ctx),
                         g[f"p{i}_binv"]) <= 1e-5


def test_transform_round_trip_large(ctx):
    import paper_1606_05688_b200 as v
    rng = np.random.default_rng(11)
    for n, pad in [((161, 150, 97), (162, 150, 98)), ((78, 80, 66), (80, 80, 70))]:
        x = rng.uniform(-1, 1, n).astype(np.float32)
        s = v.pruned_fft_forward(x, pad, ctx)
        assert rel_error(v.pruned_fft_inverse(s, pad, n, ctx), x) <= 1e-5
        b = rng.uniform(-1, 1, (2,) + n).astype(np.float32)
        sb = v.batched_fft_forward(b, pad, ctx)
        assert rel_error(v.batched_fft_inverse(sb, pad, n, ctx), b) <= 1e-5
        # nested and batched agree up to layout (fft_test.cpp:106-120)
        s0 = v.pruned_fft_forward(b[0], pad, ctx)
        zh = pad[2] // 2 + 1
        full_b = np.transpose(sb[0], (2, 1, 0))  # (px, py, zh)
        xh = pad[0] // 2 + 1
        assert rel_error(full_b[:xh, :, :zh], s0[:, :, :zh]) <= 1e-5


@pytest.mark.parametrize("mem", ["host", "device"])
def test_audited_peaks_track_the_memory_models(ctx, mem):
    """layers_test.cpp:388-414 on the device: every primitive's audited peak
    (allocator high-water mark of the call + the caller's tensors when they are
    device-resident) lies in [0.5, 1.15] x its closed-form model, and pools are
    exact (peak == model).  Shapes: the reference's (4 -> 4, k3, 8^3) plus a
    tensor-core FFT layer (80 -> 80, k5) and an f = 1 tensor-core direct layer."""
    import paper_1606_05688_b200 as v
    rng = np.random.default_rng(50)
    put = _cuda if mem == "device" else (lambda a: a)

    def band(a):
        assert a.model > 0
        assert 0.5 * a.model <= a.peak <= 1.15 * a.model, (a.peak, a.model)

    for (S, f, fo, n, k) in [(1, 4, 4, 8, 3), (2, 80, 80, 40, 5), (1, 1, 80, 60, 4)]:
        w = (rng.uniform(-1, 1, (fo, f, k, k, k)) * 0.1).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
        x = rng.uniform(-1, 1, (S, f, n, n, n)).astype(np.float32)
        p = v.ConvLayerParams(put(w), put(b), "relu")
        band(v.conv_direct(put(x), p, ctx).audit)
        band(v.conv_fft_data_parallel(put(x), p, ctx).audit)
        band(v.conv_fft_task_parallel(put(x), p, ctx).audit)
        band(v.conv_fft_staged(put(x), p, ctx).audit)
    pin = put(rng.uniform(-1, 1, (2, 3, 9, 9, 9)).astype(np.float32))
    rp = v.max_pool(pin, (3, 3, 3), ctx).audit
    band(rp)
    assert rp.peak == rp.model
    rf = v.mpf_pool(pin, (2, 2, 2), ctx).audit
    band(rf)
    assert rf.peak == rf.model


@pytest.mark.parametrize("fo", [16, 80])
def test_conv_fft_pair_tile_contraction_kept(oracle, ctx, monkeypatch, fo):
    """The earlier pair-tile tcgen05 contraction (VXG_TC_PAIR=1: 2 frequencies
    x all maps per tile, 16-byte epilogue stores) stays selectable for A/B
    timing; it must agree with the C oracle like the default quad tiles."""
    import paper_1606_05688_b200 as v
    monkeypatch.setenv("VXG_TC_PAIR", "1")
    S, f, k, T = 2, 16, (3, 2, 3), 16
    n = (T + 5, 2 * T - 3, T + 2)
    rng = np.random.default_rng(fo + 1)
    x = rng.uniform(-1, 1, (S, f) + n).astype(np.float32)
    w = (rng.uniform(-1, 1, (fo, f) + k) * np.sqrt(3.0 / (f * 18))).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
    got = v.conv_fft_tiled(x, v.ConvLayerParams(w, b, "relu"), T, tensor_cores=True, ctx=ctx)
    assert rel_error(got, oracle.conv(x, w, b, True)) <= 1e-4


@pytest.mark.parametrize("S,f,fo,n,T", [(2, 80, 80, 70, 32), (1, 16, 80, 60, 16), (1, 80, 16, 60, 16),
                                        (4, 80, 80, 40, 16), (1, 8, 16, 40, 16), (1, 80, 80, 60, 40),
                                        (2, 32, 48, 50, 36)])
def test_conv_fft_tensor_cores_match_ffma_contraction(ctx, S, f, fo, n, T):
    """The tcgen05 quad-tile contraction against the independent fp32 FFMA
    contraction on the same transforms, at sizes where every CTA loops over
    many tiles and both shared-memory rings wrap many times (a cross-proxy
    race in the staged-X ring showed only here), incl. the pair-only T = 36/40."""
    import torch
    import paper_1606_05688_b200 as v
    g = torch.Generator(device="cuda").manual_seed(S * 1000 + f + fo + n + T)
    x = torch.rand((S, f, n, n, n), device="cuda", generator=g) * 2 - 1
    w = (torch.rand((fo, f, 5, 5, 5), device="cuda", generator=g) * 2 - 1) * (3.0 / (f * 125)) ** 0.5
    b = (torch.rand((fo,), device="cuda", generator=g) * 2 - 1) * 0.1
    p = v.ConvLayerParams(w.contiguous(), b.contiguous(), "identity")
    a = v.conv_fft_tiled(x, p, T, tensor_cores=False, ctx=ctx)
    c = v.conv_fft_tiled(x, p, T, tensor_cores=True, ctx=ctx)
    err = ((a - c).abs().max() / a.abs().max()).item()
    assert err <= 1e-5, err


@pytest.mark.parametrize("T", [24, 32])
def test_conv_fft_fused_z_load_vs_oracle(oracle, ctx, T):
    """The CTA-pair forward transform's fused path (interior boxes with 16-byte
    aligned z rows load their rows straight into registers for the z r2c):
    z extent a multiple of 4 and V = T - 4 a multiple of 4 select it, boundary
    boxes take the staged path -- both against the C oracle."""
    import paper_1606_05688_b200 as v
    S, f, fo, k = 2, 16, 16, (5, 5, 5)
    n = (2 * (T - 4) + 9, 2 * (T - 4) + 6, 3 * (T - 4) + 4)
    assert n[2] % 4 == 0
    rng = np.random.default_rng(T)
    x = rng.uniform(-1, 1, (S, f) + n).astype(np.float32)
    w = (rng.uniform(-1, 1, (fo, f) + k) * np.sqrt(3.0 / (f * 125))).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
    got = v.conv_fft_tiled(_cuda(x), v.ConvLayerParams(_cuda(w), _cuda(b), "relu"), T, tensor_cores=True,
                           cta_pair=True, ctx=ctx)
    assert rel_error(got.cpu().numpy(), oracle.conv(x, w, b, True)) <= 1e-4


@pytest.mark.parametrize("fo", [32, 80])
def test_conv_fft_quad_tiles_3xtf32_split(oracle, ctx, monkeypatch, fo):
    """The quad-tile contraction with the 3xTF32 split (VXG_Q_3TF32=1: three tf32
    MMAs per product instead of tf32 + one bf16 correction MMA; the W layout
    follows the same switch) against the C oracle."""
    import paper_1606_05688_b200 as v
    monkeypatch.setenv("VXG_Q_3TF32", "1")
    S, f, k, T = 2, 16, (3, 3, 3), 16
    n = (T + 9, 2 * T - 1, T + 4)
    rng = np.random.default_rng(fo + 7)
    x = rng.uniform(-1, 1, (S, f) + n).astype(np.float32)
    w = (rng.uniform(-1, 1, (fo, f) + k) * np.sqrt(3.0 / (f * 27))).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
    got = v.conv_fft_tiled(x, v.ConvLayerParams(w, b, "relu"), T, tensor_cores=True, ctx=ctx)
    assert rel_error(got, oracle.conv(x, w, b, True)) <= 1e-4


@pytest.mark.parametrize("T,pair", [(24, True), (32, True), (40, True), (8, False), (16, False),
                                    (32, False), (36, False)])
def test_conv_fft_single_input_map_fused_inverse(oracle, ctx, T, pair):
    """f = 1 FFT layers (the first layers of n726/n926) skip the Y spectra: the
    inverse (CTA pair or one CTA) multiplies each input spectrum line by its
    output map's kernel spectrum on load.  Against the C oracle, several tiles
    per axis."""
    import paper_1606_05688_b200 as v
    S, f, fo, k = 2, 1, 16, (min(7, T), min(6, T), min(5, T))
    n = (2 * T + 3, T + 8, 2 * T - 5)
    rng = np.random.default_rng(T + 100)
    x = rng.uniform(-1, 1, (S, f) + n).astype(np.float32)
    w = (rng.uniform(-1, 1, (fo, f) + k) * 0.1).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
    got = v.conv_fft_tiled(x, v.ConvLayerParams(w, b, "relu"), T, tensor_cores=False, cta_pair=pair, ctx=ctx)
    assert rel_error(got, oracle.conv(x, w, b, True)) <= 1e-4


@pytest.mark.parametrize("mem", ["host", "device"])
def test_mpf_rejects_nan_anywhere(ctx, mem):
    """mpf_pool rejects a NaN wherever it sits (layers.hpp:429): the 2x2x2 kernel
    checks the values its windows read, so every position class -- corners,
    faces, the last plane of each axis, tile seams of its 16 x 8 x 64 staging --
    must still be caught."""
    import paper_1606_05688_b200 as v
    n = (35, 19, 131)
    rng = np.random.default_rng(9)
    base = rng.uniform(-1, 1, (2, 3) + n).astype(np.float32)
    put = _cuda if mem == "device" else (lambda a: a)
    assert v.mpf_pool(put(base), (2, 2, 2), ctx).output is not None
    for pos in [(0, 0, 0, 0, 0), (1, 2, 34, 18, 130), (0, 1, 34, 0, 0), (0, 0, 0, 18, 0), (1, 0, 0, 0, 130),
                (0, 2, 16, 8, 64), (1, 1, 15, 7, 63), (0, 0, 17, 9, 65), (1, 2, 33, 17, 129)]:
        x = base.copy()
        x[pos] = np.nan
        with pytest.raises(ValueError, match="NaN"):
            v.mpf_pool(put(x), (2, 2, 2), ctx)
    v.mpf_pool(put(base), (2, 2, 2), ctx)  # the flag was cleared




def test_conv_fft_quad_tiles_short_layers(oracle, ctx):
    """The quad contraction on layers with fewer than 128 spectrum rows (its X
    boxes then cover only the rows the tensor has) and with the widest map
    count, against the C oracle."""
    import paper_1606_05688_b200 as v
    rng = np.random.default_rng(41)
    for S, f, fo, T in ((2, 24, 32, 16), (1, 16, 80, 24)):
        k = (3, 3, 3)
        n = (T + 9, 2 * T - 1, T + 4) if S > 1 else (T + 2,) * 3
        x = rng.uniform(-1, 1, (S, f) + n).astype(np.float32)
        w = (rng.uniform(-1, 1, (fo, f) + k) * np.sqrt(3.0 / (f * 27))).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
        got = v.conv_fft_tiled(x, v.ConvLayerParams(w, b, "relu"), T, tensor_cores=True, ctx=ctx)
        assert rel_error(got, oracle.conv(x, w, b, True)) <= 1e-4, (S, f, fo, T)
