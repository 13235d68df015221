"""Halo-tiled dense inference of a large volume across ranks.

The paper's overlap-save patches with no reference code:
the dense output (extent V - fov + 1 per axis) is cut into tiles whose output
extent is a multiple of the MPF stride product; each tile's input crop is its
output box plus a halo of fov - 1.  Tiles are independent (translation
equivariance), so ranks process disjoint tile sets with no data-path
collective; the last tile along an axis shifts inward instead of padding, and
only the part of it no earlier tile wrote is stored.  Outputs are idempotent
per tile, which makes resume trivial (``done`` set).  An optional gather
brings every rank's tiles to rank 0 over torch.distributed (NCCL over
NVLink on GPUs, gloo on CPU).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass
from typing import Callable, Iterable, Optional, Sequence

import numpy as np


@dataclass(frozen=True)
class Tile:
    index: int
    out_origin: tuple       # dense-output coordinates of the tile's output box
    out_extent: tuple
    in_origin: tuple        # input coordinates of the crop (= out_origin)
    in_extent: tuple        # out_extent + fov - 1
    write_origin: tuple     # the part of the output box this tile owns
    write_extent: tuple


def _axis_tiles(dense: int, tile: int):
    """[(origin, write_origin, write_extent)] along one axis."""
    if tile >= dense:
        return [(0, 0, dense)]
    out = []
    o = 0
    while o + tile < dense:
        out.append((o, o, tile))
        o += tile
    last = dense - tile  # shifted inward: same extent, overlap is recomputed, not rewritten
    out.append((last, o, dense - o))
    return out


def plan_tiles(volume: Sequence[int], fov: Sequence[int], tile_out: Sequence[int],
               align: Sequence[int] = (1, 1, 1)) -> list:
    dense = [int(volume[a]) - int(fov[a]) + 1 for a in range(3)]
    if any(d <= 0 for d in dense):
        raise ValueError("tiler: volume smaller than the field of view")
    ext = []
    for a in range(3):
        # a tile's crop is admissible only if its output extent is a multiple of
        # the MPF stride product; a dense extent that is not gets a shifted last tile
        t = min(int(tile_out[a]), dense[a])
        t -= t % align[a]
        if t <= 0:
            raise ValueError("tiler: tile extent incompatible with the MPF stride")
        ext.append(t)
    axes = [_axis_tiles(dense[a], ext[a]) for a in range(3)]
    tiles = []
    for i, (ax, ay, az) in enumerate(itertools.product(*axes)):
        o = (ax[0], ay[0], az[0])
        e = tuple(min(ext[a], dense[a]) for a in range(3))
        tiles.append(Tile(i, o, e, o, tuple(e[a] + int(fov[a]) - 1 for a in range(3)),
                          (ax[1], ay[1], az[1]), (ax[2], ay[2], az[2])))
    return tiles


def assign(tiles: Sequence[Tile], rank: int, world: int) -> list:
    """Static round-robin (tile i -> rank i % world)."""
    return [t for t in tiles if t.index % world == rank]


def run_tiles(forward: Callable, volume, tiles: Iterable[Tile], out=None,
              done: Optional[set] = None, forward_many: Optional[Callable] = None, batch: int = 4):
    """forward(crop (1, f, *in_extent)) -> (1, f_out, *out_extent) array.
    Writes each tile's owned region into `out` (dense, (1, f_out, *dense)) if
    given; returns {tile index: owned block}.  Tiles in `done` are skipped.
    forward_many(list of crops) -> list of results (optional): tiles of one
    extent then run `batch` at a time through it, so uploads and downloads of
    neighbouring tiles overlap the forwards."""
    blocks = {}
    todo = [t for t in tiles if not (done is not None and t.index in done)]

    def crop_of(t):
        sl = tuple(slice(t.in_origin[a], t.in_origin[a] + t.in_extent[a]) for a in range(3))
        return np.ascontiguousarray(volume[(slice(None), slice(None)) + sl], dtype=np.float32)

    results = {}
    if forward_many is not None:
        for b0 in range(0, len(todo), batch):
            grp = todo[b0:b0 + batch]
            same = all(t.in_extent == grp[0].in_extent for t in grp)
            outs = forward_many([crop_of(t) for t in grp]) if same else [forward(crop_of(t)) for t in grp]
            for t, r in zip(grp, outs):
                results[t.index] = r
    for t in todo:
        res = np.asarray(results.pop(t.index)) if t.index in results else np.asarray(forward(crop_of(t)))
        rel = tuple(slice(t.write_origin[a] - t.out_origin[a],
                          t.write_origin[a] - t.out_origin[a] + t.write_extent[a]) for a in range(3))
        block = res[(slice(None), slice(None)) + rel]
        if out is not None:
            dst = tuple(slice(t.write_origin[a], t.write_origin[a] + t.write_extent[a])
                        for a in range(3))
            out[(slice(None), slice(None)) + dst] = block
        blocks[t.index] = block
        if done is not None:
            done.add(t.index)
    return blocks


def gather_to_root(blocks: dict, tiles: Sequence[Tile], out, f_out: int, device="cpu"):
    """Rank r sends its owned blocks to rank 0 (torch.distributed point-to-point;
    NCCL over NVLink when device is CUDA).  Rank 0 writes them into `out`."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    for t in tiles:
        owner = t.index % world
        shape = (1, f_out) + tuple(t.write_extent)
        if owner == 0:
            continue
        if rank == owner:
            dist.send(torch.from_numpy(np.ascontiguousarray(blocks[t.index])).to(device), dst=0)
        elif rank == 0:
            buf = torch.empty(shape, dtype=torch.float32, device=device)
            dist.recv(buf, src=owner)
            dst = tuple(slice(t.write_origin[a], t.write_origin[a] + t.write_extent[a])
                        for a in range(3))
            out[(slice(None), slice(None)) + dst] = buf.cpu().numpy()
    if rank == 0:
        for t in tiles:
            if t.index % world == 0:
                dst = tuple(slice(t.write_origin[a], t.write_origin[a] + t.write_extent[a])
                            for a in range(3))
                out[(slice(None), slice(None)) + dst] = blocks[t.index]


def infer_volume(model, volume, tile_out, rank: int = 0, world: int = 1, gather: bool = True,
                 done: Optional[set] = None):
    """Dense inference of `volume` (1, f_in, X, Y, Z) with a vxg Model, tiles
    distributed round-robin over ranks.  Returns the dense output on rank 0
    (gathered) or this rank's blocks."""
    fov = model.net.field_of_view()
    align = [1, 1, 1]
    for l in model.net.layers:
        if l[0] == "pool":
            align = [align[a] * l[1][a] for a in range(3)]
    tiles = plan_tiles(volume.shape[2:], fov, tile_out, align)
    mine = assign(tiles, rank, world)
    dense = tuple(int(volume.shape[2 + a]) - fov[a] + 1 for a in range(3))
    out = np.zeros((1, model.net.features_out) + dense, np.float32) if (rank == 0 or world == 1) else None

    def fwd(crop):
        res, _ = model.forward(np.ascontiguousarray(crop, np.float32))
        return res

    def fwd_many(crops):
        res, _ = model.forward_many(crops)
        return res

    blocks = run_tiles(fwd, volume, mine, out if world == 1 else None, done,
                       forward_many=fwd_many if hasattr(model, "forward_many") else None)
    if world > 1 and gather:
        gather_to_root(blocks, tiles, out, model.net.features_out,
                       device="cuda" if _cuda_dist() else "cpu")
    return out if (rank == 0 or world == 1) else blocks


def _cuda_dist() -> bool:
    import torch.distributed as dist
    return dist.get_backend() == "nccl"
