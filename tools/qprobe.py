"""Quad contraction probe: tensor-core tiled FFT conv vs the FFMA contraction
(GPU vs GPU) over map counts and row counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1606_05688_b200 as v
ctx = v.Context(0)
g = torch.Generator(device="cuda").manual_seed(3)
for (S, f, fo, n, T) in [(1, 80, 80, 40, 16), (2, 80, 80, 70, 32), (1, 16, 80, 60, 16), (1, 80, 16, 60, 16),
                         (2, 24, 32, 50, 24), (4, 80, 80, 40, 16), (1, 8, 16, 40, 16)]:
    x = torch.rand((S, f, n, n, n), device="cuda", generator=g) * 2 - 1
    w = (torch.rand((fo, f, 5, 5, 5), device="cuda", generator=g) * 2 - 1) * (3.0 / (f * 125)) ** 0.5
    b = (torch.rand((fo,), device="cuda", generator=g) * 2 - 1) * 0.1
    p = v.ConvLayerParams(w.contiguous(), b.contiguous(), "identity")
    a = v.conv_fft_tiled(x, p, T, tensor_cores=False, ctx=ctx)
    c = v.conv_fft_tiled(x, p, T, tensor_cores=True, ctx=ctx)
    err = ((a - c).abs().max() / a.abs().max()).item()
    d = (a - c).abs().reshape(S, fo, -1).amax(dim=2)
    bad = (d > 1e-4 * a.abs().max()).nonzero()
    print(S, f, fo, n, T, "err", err, "bad (s,map) count", len(bad), bad[:8].tolist(), flush=True)
