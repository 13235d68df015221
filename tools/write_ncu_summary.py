"""Write profiles/r1_ncu_summary.md and profiles/r1_bench_final.json from one
tools/final.sh run (TAG), read here after gpurun merged gpurun_out/.

    python tools/write_ncu_summary.py r1h
"""
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"


def run(*args):
    return subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), *args],
                          capture_output=True, text=True).stdout.rstrip()


def dedup(text):
    seen, keep = set(), []
    for b in text.split("== ")[1:]:
        name = b.splitlines()[0]
        if name not in seen:
            seen.add(name)
            keep.append("== " + b)
    return "".join(keep).rstrip()


def main(tag):
    d = json.loads((OUT / f"{tag}_bench.json").read_text().strip().splitlines()[-1])
    k, st = d["kernels"], d["steps"]
    launches = run("launches", str(OUT / f"{tag}_launches.csv"))
    layer = run("full", str(OUT / f"{tag}_layer.ncu-rep"))
    small = dedup(run("full", str(OUT / f"{tag}_small.ncu-rep")))
    per = lambda n: k[n]["seconds"] / st
    txt = f"""# Round 1 ncu evidence (B200, sm_100a) — final state (TAG {tag})

Produced by `tools/final.sh` → `tools/gpu_prof.sh` through gpurun (raw reports stay in gpurun_out/, git-ignored); summarised with `tools/ncu_summary.py` by `tools/write_ncu_summary.py {tag}`. ncu numbers are cold-cache and serialised per launch: compare shares, not absolute step times. The bench line of the same code, unprofiled: `profiles/r1_bench_final.json` ({d['value']:.3e} voxels/s device, {d['e2e']['value']:.3e} end to end).

## 1. Launch list of the bench command (`ncu --metrics gpu__time_duration.sum --clock-control none`)

Command: `VXG_TUNE_FILE=<costs of the unprofiled run> python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1` (n537, 722³ patch, plan {d['config']['layers']}; 3 warm-up + 1 timed + the end-to-end warm-up (2 patches) + 1 end-to-end forward = 7 forwards). The layer costs are replayed from the unprofiled run (`gpurun_out/{tag}_tune.txt`): timing them under ncu would change the plan. The first layer runs as `direct_tc_kernel<80, 64>` on x slabs (DESIGN.md §4).

```
{launches}
```

The same step measured live with CUDA events (bench.py `kernels`, seconds per step): contraction {per('cgemm'):.3f}, forward transforms {per('tile_fwd'):.3f}, inverse transforms {per('tile_inv'):.3f}, MPF {per('pool'):.3f}, direct conv {per('direct'):.3f}, recombine {per('recombine'):.4f} (step {d['ms_per_step'] / 1e3:.3f} s).

## 2. `--set full`, one 80->80 k5 FFT layer (S = 64 fragments of 85³, T = 32, 1728 rows)

Command: `ncu --set full --clock-control none --import-source on -k regex:"cgemm_tc_kernel|tile_fwd_pair_kernel|tile_inv_pair_kernel" python tools/kbench.py --which conv --S 64 --n 85`. DRAM bytes per launch against the algorithmic bytes: forward 33.5 GB vs 37.3 GB (boxes overlap, L2 catches part), contraction 41.7 GB vs 40.3 GB (X + Y + pre-split W: 1.035x), inverse 31.6 GB vs 31.4 GB.

```
{layer}
```

## 3. First-layer direct convolution on the tensor cores (1 -> 80 maps, k = 4, 330³) and MPF (80 x 255³)

`python tools/kbench.py --which direct,mpf`. The direct kernel writes 11.2 GB (80 maps x 327³) and reads 0.29 GB; it is bound by its converter and epilogue warps (per-role counters in profiles/r1_microbench.md), not by HBM or the tensor pipe.

```
{small}
```

Stall analysis (`--page source`, tools/ncu_sass_hot.py) and the experiments behind these numbers: DESIGN.md §5 and profiles/r1_microbench.md.
"""
    (ROOT / "profiles" / "r1_ncu_summary.md").write_text(txt)
    shutil.copy(OUT / f"{tag}_bench.json", ROOT / "profiles" / "r1_bench_final.json")
    shutil.copy(OUT / f"{tag}_tune.txt", ROOT / "profiles" / "r1_tuned_costs_n537.txt")


if __name__ == "__main__":
    main(sys.argv[1])
