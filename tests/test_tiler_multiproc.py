"""CPU: the N>1 host logic -- halo tiling, round-robin rank assignment, resume,
and the point-to-point gather to rank 0 -- across world_size 2 with the gloo
backend.  A numpy stand-in with a known field of view replaces the network
(the tiler only relies on translation equivariance)."""
import os
import socket

import numpy as np
import pytest

from paper_1606_05688_b200 import tiler


def box_net(x, fov):
    """dense out[d] = sum(in[d : d + fov]) per axis (a translation-equivariant 'net')."""
    c = np.cumsum(np.cumsum(np.cumsum(x, axis=2), axis=3), axis=4)
    c = np.pad(c, ((0, 0), (0, 0), (1, 0), (1, 0), (1, 0)))
    f = fov
    s = (c[:, :, f:, f:, f:] - c[:, :, :-f, f:, f:] - c[:, :, f:, :-f, f:] - c[:, :, f:, f:, :-f]
         + c[:, :, :-f, :-f, f:] + c[:, :, :-f, f:, :-f] + c[:, :, f:, :-f, :-f]
         - c[:, :, :-f, :-f, :-f])
    return s.astype(np.float32)


def test_plan_tiles_cover_output_exactly_once():
    vol, fov = (50, 41, 37), (7, 7, 7)
    tiles = tiler.plan_tiles(vol, fov, (16, 16, 16), (4, 4, 4))
    dense = [vol[a] - fov[a] + 1 for a in range(3)]
    cover = np.zeros(dense, np.int32)
    for t in tiles:
        assert all(t.in_extent[a] == t.out_extent[a] + fov[a] - 1 for a in range(3))
        assert all(e % 4 == 0 for e in t.out_extent)
        assert all(t.in_origin[a] + t.in_extent[a] <= vol[a] for a in range(3))
        sl = tuple(slice(t.write_origin[a], t.write_origin[a] + t.write_extent[a]) for a in range(3))
        cover[sl] += 1
    assert (cover == 1).all()
    mine = [tiler.assign(tiles, r, 3) for r in range(3)]
    assert sorted(t.index for m in mine for t in m) == list(range(len(tiles)))


def test_plan_tiles_tile_larger_than_unaligned_dense():
    """tile_out >= dense with dense % align != 0: the tile shrinks to
    the largest aligned extent and a shifted last tile covers the rest."""
    vol, fov = (30, 29, 28), (7, 7, 7)  # dense 24, 23, 22
    tiles = tiler.plan_tiles(vol, fov, (64, 64, 64), (4, 4, 4))
    dense = [vol[a] - fov[a] + 1 for a in range(3)]
    cover = np.zeros(dense, np.int32)
    for t in tiles:
        assert all(e % 4 == 0 for e in t.out_extent)
        assert all(t.in_origin[a] + t.in_extent[a] <= vol[a] for a in range(3))
        sl = tuple(slice(t.write_origin[a], t.write_origin[a] + t.write_extent[a]) for a in range(3))
        cover[sl] += 1
    assert (cover == 1).all()
    assert [t.out_extent for t in tiles][0] == (24, 20, 20)


def test_run_tiles_batched_streaming_path():
    """The forward_many path (batches of equal-extent tiles) writes exactly what
    the one-tile path writes, and still honours resume."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, 2, 41, 35, 30)).astype(np.float32)
    fov = 5
    full = box_net(x, fov)
    tiles = tiler.plan_tiles(x.shape[2:], (fov,) * 3, (10, 12, 9))
    batches = []

    def many(crops):
        batches.append(len(crops))
        return [box_net(c, fov) for c in crops]

    out = np.zeros_like(full)
    done = {tiles[0].index}
    out_first = np.zeros_like(full)
    tiler.run_tiles(lambda c: box_net(c, fov), x, tiles[:1], out_first)
    out += out_first
    tiler.run_tiles(lambda c: box_net(c, fov), x, tiles, out, done, forward_many=many, batch=3)
    assert sum(batches) == len(tiles) - 1 and max(batches) == 3
    np.testing.assert_allclose(out, full, rtol=1e-4, atol=1e-3)  # fp32 cumsums of crops vs volume


def test_run_tiles_matches_full_and_resumes():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((1, 2, 40, 33, 29)).astype(np.float32)
    fov = 6
    full = box_net(x, fov)
    tiles = tiler.plan_tiles(x.shape[2:], (fov,) * 3, (12, 12, 12))
    out = np.zeros_like(full)
    done = set()
    tiler.run_tiles(lambda c: box_net(c, fov), x, tiles[: len(tiles) // 2], out, done)
    calls = []

    def counting(c):
        calls.append(1)
        return box_net(c, fov)

    tiler.run_tiles(counting, x, tiles, out, done)  # resume: finished tiles are skipped
    assert len(calls) == len(tiles) - len(tiles) // 2
    np.testing.assert_allclose(out, full, rtol=1e-5, atol=1e-4)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((1, 1, 36, 30, 34)).astype(np.float32)
    fov = 5
    tiles = tiler.plan_tiles(x.shape[2:], (fov,) * 3, (8, 8, 8), (2, 2, 2))
    mine = tiler.assign(tiles, rank, world)
    blocks = tiler.run_tiles(lambda c: box_net(c, fov), x, mine)
    dense = tuple(x.shape[2 + a] - fov + 1 for a in range(3))
    out = np.zeros((1, 1) + dense, np.float32) if rank == 0 else None
    tiler.gather_to_root(blocks, tiles, out, 1, device="cpu")
    # timing reduction of the bench: max over ranks
    import torch
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((np.abs(out - box_net(x, fov)).max(), t.item(), len(mine)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_gloo():
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    err, tmax, n0 = q.get(timeout=10)
    assert err < 1e-3
    assert tmax == 2.0
    assert n0 > 0


def test_bench_self_launches_n_ranks():
    """`python bench.py --gpus 2` (no torchrun, no WORLD_SIZE) re-runs itself
    under torch.distributed.run with 2 ranks; the line reports n_gpus 2 and the
    whole-job value = ranks x steps x voxels / max-over-ranks time (the --stub
    step keeps it on CPU / gloo)."""
    import json
    import subprocess
    import sys
    from conftest import ROOT
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--stub", "--steps", "3",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["steps"] == 3
    assert d["value"] == pytest.approx(2 * 3 * d["voxels_per_rank_step"] / d["elapsed_max_over_ranks"])


def test_synthetic_volume_crops_are_consistent():
    """SyntheticVolume (counter-based, C5's 2048^3 input without 34 GB of host
    memory): any crop equals the same window of the materialised volume, values
    in [-1, 1), reproducible per seed."""
    v = tiler.SyntheticVolume((1, 2, 9, 11, 13), seed=3)
    full = v[:, :, 0:9, 0:11, 0:13]
    assert full.shape == (1, 2, 9, 11, 13) and full.dtype == np.float32
    assert full.min() >= -1.0 and full.max() < 1.0 and abs(float(full.mean())) < 0.2
    np.testing.assert_array_equal(v[:, 1:2, 2:7, 3:11, 5:6], full[:, 1:2, 2:7, 3:11, 5:6])
    assert not np.array_equal(tiler.SyntheticVolume((1, 2, 9, 11, 13), seed=4)[:, :, 0:9, 0:11, 0:13], full)


def _worker_shared(rank, world, port, path, q):
    """Both ranks read one memmapped input file and write their tiles into one
    shared output memmap (no per-rank copy of the volume, no gather)."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = np.load(path + ".in.npy", mmap_mode="r")
    fov = 5
    tiles = tiler.plan_tiles(x.shape[2:], (fov,) * 3, (8, 8, 8), (2, 2, 2))
    dense = tuple(x.shape[2 + a] - fov + 1 for a in range(3))
    out = tiler.open_shared_output(path + ".out.npy", (1, 1) + dense, rank, world)
    timings = []
    tiler.run_tiles(lambda c: box_net(c, fov), x, tiler.assign(tiles, rank, world), out,
                    timings=timings, keep_blocks=False)
    out.flush()
    dist.barrier()
    if rank == 0:
        q.put((np.abs(np.load(path + ".out.npy") - box_net(np.asarray(x), fov)).max(), len(timings)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shared_memmap_output_gloo(tmp_path):
    import torch.multiprocessing as mp
    rng = np.random.default_rng(2)
    path = str(tmp_path / "vol")
    np.save(path + ".in.npy", rng.standard_normal((1, 1, 36, 30, 34)).astype(np.float32))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_shared, args=(r, 2, port, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    err, nbatches = q.get(timeout=10)
    assert err < 1e-3 and nbatches > 0
