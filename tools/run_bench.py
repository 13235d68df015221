"""Device counterpart of the reference's `voxinfer bench` (proj/src/cli.cpp:225-280):
sweep the admissible cubic input extents of a net, run one forward per extent
with the measured-time planner, and write the same CSV

    input_extent,memory_model,memory_audited,voxels_per_sec,seconds,layer0_ms,...

memory_model = the planner's peak (scalars = bytes / 4, the reference's unit) for the extent (vxg_model_plan_bytes,
the reference's host_peak + device_peak model column), memory_audited = the
allocator high-water mark of the forward (ThroughputReport.device_peak), seconds
/ layerN_ms = CUDA-event times of the forward (execute.hpp:228-239).  Input per
extent: fill_random(seed ^ (0x9e3779b97f4a7c15 * e)) as cli.cpp:261; weights
random_weights(net, seed) as cli.cpp:246.  Extents that do not fit the HBM budget
are skipped with a note, like the reference's resource_exhausted rows.

    python tools/run_bench.py --net n537 --min-extent 170 --max-extent 738 --every 64 [--csv out.csv]
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402


def admissible(net, e: int) -> bool:
    """Every layer's shape is valid at extent e with all pools as MPF (the
    reference planner's fragment plan, planner.cpp:536-589)."""
    if e < max(net.field_of_view()):
        return False
    _, viol = net.propagate(1, (e, e, e))
    return viol < 0


def main(argv=None) -> int:
    import torch

    import paper_1606_05688_b200 as v
    from paper_1606_05688_b200.bundled_nets import NETS

    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="n537")
    ap.add_argument("--net-file", default="", help="a .net description instead of a bundled net")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--min-extent", type=int, default=0, help="default: the field of view")
    ap.add_argument("--max-extent", type=int, default=0, help="default: min-extent + 64")
    ap.add_argument("--every", type=int, default=1, help="keep every k-th admissible extent")
    ap.add_argument("--csv", default="", help="write rows here (default: stdout)")
    ap.add_argument("--no-tune", action="store_true", help="modelled instead of measured layer costs")
    a = ap.parse_args(argv)

    text = Path(a.net_file).read_text() if a.net_file else NETS[a.net]
    net = v.parse_network_spec(text)
    fov = max(net.field_of_view())
    lo = a.min_extent or fov
    hi = a.max_extent or lo + 64
    ctx = v.Context(0)
    model = v.Model(net, v.random_weights(net, a.seed), ctx)
    # the context budget, capped by what the device has free now (another
    # context or torch's cache in the same process may hold memory outside it)
    torch.cuda.empty_cache()
    ctx.trim()
    budget = min(ctx.memory()["budget"] - ctx.memory()["current"], torch.cuda.mem_get_info()[0] - (2 << 30))
    out = open(a.csv, "w") if a.csv else sys.stdout
    note = sys.stdout if a.csv else sys.stderr  # cli.cpp:235: notes beside the rows
    note.write(f"seed {a.seed}\n")
    out.write("input_extent,memory_model,memory_audited,voxels_per_sec,seconds"
              + "".join(f",layer{i}_ms" for i in range(net.layer_count)) + "\n")
    rows, k = 0, 0
    for e in range(lo, hi + 1):
        if not admissible(net, e):
            continue
        k += 1
        if (k - 1) % a.every:
            continue
        need = model.plan_bytes(1, e)
        dense = 4 * (e ** 3) + 4 * net.features_out * (e - fov + 1) ** 3
        if need <= 0 or need + dense > budget:
            note.write(f"extent {e}: skipped (plan needs {need + dense} bytes, budget {budget})\n")
            continue
        if not a.no_tune:
            model.tune(1, e)
        seed = (a.seed ^ ((0x9E3779B97F4A7C15 * e) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF
        x = torch.from_numpy(v.fill_random((1, net.features_in, e, e, e), seed)).cuda()
        ctx.reset_peak()
        try:
            y, rep = model.forward(x, cache_spectra=False)
        except v.ResourceExhausted as ex:
            note.write(f"extent {e}: skipped ({ex})\n")
            continue
        del y, x
        out.write(f"{e},{need // 4},{int(rep.device_peak)},{rep.voxels_per_second:.12g},{rep.seconds:.12g}"
                  + "".join(f",{s * 1e3:.12g}" for s in rep.layer_seconds) + "\n")
        out.flush()
        rows += 1
    model.close()
    if a.csv:
        out.close()
        print(f"wrote {rows} rows to {a.csv}")
    if rows == 0:
        sys.stderr.write(f"infeasible: no admissible input extent in [{lo}, {hi}]\n")
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
