#!/usr/bin/env python
"""C5: n537 dense inference of a 2048^3 volume in halo tiles
of 634^3 -> 472^3 (4^3 = 64 tiles; the last tile per axis shifts 2 voxels
inward), through paper_1606_05688_b200.tiler.infer_volume -- the multi-GPU
path's unit of work, here at N = 1 (or as one rank of N under torchrun).

The input is a SyntheticVolume (counter-based generator, crops made on the GPU
and handed over as host arrays, as a volume file would be); the output is one
shared .npy memmap every rank writes its tiles into.  Prints one JSON line:
tiles run, seconds, per-tile times (crop / forward incl. H2D + D2H / write),
voxels/s, and a parity spot check (an 8^3 block of the tiled output against a
single forward of the matching 170^3 input crop).

    python tools/c5_volume.py [--tiles 8] [--out /tmp/c5_out.npy] [--batch 4]
    torchrun --nproc-per-node N tools/c5_volume.py --tiles 64
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--volume", type=int, default=2048)
    ap.add_argument("--tile-in", type=int, default=634)
    ap.add_argument("--tiles", type=int, default=8, help="run the first K tiles (0: all)")
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--out", default="/tmp/c5_out.npy")
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1606_05688_b200 as v
    from paper_1606_05688_b200 import tiler
    from paper_1606_05688_b200.bundled_nets import FOV, NETS

    net = v.parse_network_spec(NETS["n537"])
    fov = FOV["n537"]
    ctx = v.Context(local)
    model = v.Model(net, v.random_weights(net, 1), ctx)
    e = args.tile_in
    t0 = time.perf_counter()
    model.tune(1, e)
    cands = [None, ["direct"] + ["auto"] * (net.conv_count - 1)]
    algos = min(cands, key=lambda a: sum(l["seconds"] for l in model.plan_info(1, e, a)))
    t_tune = time.perf_counter() - t0

    class Planned:
        """the Model with the chosen per-layer algorithms (infer_volume's model)"""
        def __init__(self, m):
            self.m, self.net = m, m.net

        def forward(self, x):
            return self.m.forward(x, conv_algos=algos)

        def forward_many(self, xs):
            return self.m.forward_many(xs, conv_algos=algos)

    vol = tiler.SyntheticVolume((1, 1) + (args.volume,) * 3, seed=1, device="cuda")
    tile_out = e - fov + 1
    all_tiles = tiler.plan_tiles(vol.shape[2:], (fov,) * 3, (tile_out,) * 3, (8, 8, 8))
    subset = [t.index for t in all_tiles][: args.tiles or len(all_tiles)]
    timings = []
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    out = tiler.infer_volume(Planned(model), vol, (tile_out,) * 3, rank=rank, world=ws, out_path=args.out,
                             batch=args.batch, timings=timings, tile_subset=subset)
    elapsed = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    mine = [t for t in all_tiles if t.index in set(subset) and t.index % ws == rank]
    owned = sum(int(np.prod(t.write_extent)) for t in mine)
    computed = len(subset) * tile_out ** 3  # every tile computes a full 472^3 output box
    # parity spot check: an 8^3 block of the tiled output vs one forward of the
    # matching 170^3 crop (translation equivariance), on rank 0's first tile
    check = None
    if rank == 0 and mine:
        t = mine[0]
        o = [t.write_origin[a] + 17 for a in range(3)]
        crop = vol[(slice(None), slice(None)) + tuple(slice(o[a], o[a] + 170) for a in range(3))]
        want, _ = model.forward(np.ascontiguousarray(crop), conv_algos=algos)
        got = np.asarray(out[(slice(None), slice(None)) + tuple(slice(o[a], o[a] + 8) for a in range(3))])
        check = {"tile": t.index, "origin": o,
                 "rel_err": float(np.abs(got - want).max() / np.abs(want).max())}
    per_tile = [r["forward_s"] / len(r["tiles"]) for r in timings]
    line = {
        "metric": "output voxels/sec, n537 2048^3 volume in halo tiles (C5)", "n_gpus": ws,
        "volume": args.volume, "tile_in": e, "tile_out": tile_out, "tiles_total": len(all_tiles),
        "tiles_run": len(subset), "seconds": elapsed,
        "value": computed / elapsed,  # output voxels computed per second, all ranks
        "owned_voxels_per_s": owned * ws / elapsed,
        "unit": "voxels/s", "plan": [l.get("algo", "mpf") for l in model.plan_info(1, e, algos)],
        "tune_s": t_tune, "per_tile_forward_s": per_tile,
        "crop_s": sum(r["crop_s"] for r in timings), "forward_s": sum(r["forward_s"] for r in timings),
        "write_s": sum(r["write_s"] for r in timings),
        "extrapolated_full_volume_s_1gpu": elapsed / len(subset) * len(all_tiles) * ws,
        "parity_vs_single_patch": check,
        "input": "SyntheticVolume (splitmix64 counter-based, crops generated on the GPU, handed over as host "
                 "arrays); output: shared .npy memmap",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    model.close()
    ctx.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
