"""Summaries of ncu outputs for profiles/ (read here, after gpurun):

    python tools/ncu_summary.py launches <launches.csv>     per-kernel launch totals
    python tools/ncu_summary.py full <report.ncu-rep>        key --set full metrics per kernel
"""
import collections
import csv
import io
import subprocess
import sys


def fl(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return 0.0


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "").replace("vxg::", "")
        agg[name][0] += 1
        agg[name][1] += fl(r[vi])
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':36s} {'launches':>8s} {'total ms':>10s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:36s} {n:8d} {t / 1e6:10.2f} {100 * t / tot:5.1f}%")
    print(f"{'(all)':36s} {sum(a[0] for a in agg.values()):8d} {tot / 1e6:10.2f}")


METRICS = [
    ("gpu__time_duration.sum", "duration", 1e-3, "ms"),
    ("dram__bytes_read.sum", "DRAM read", 1.0, "GB?"),
    ("dram__bytes_write.sum", "DRAM write", 1.0, "GB?"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak", 1.0, "%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak", 1.0, "%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 % peak", 1.0, "%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak", 1.0, "%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1.0, "%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %", 1.0, "%"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe %", 1.0, "%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %", 1.0, "%"),
    ("launch__registers_per_thread", "registers", 1.0, ""),
    ("launch__grid_size", "grid", 1.0, ""),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1.0, "%"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        print(f"== {name[:90]}")
        for key, label, _, _ in METRICS:
            if key in h:
                i = h.index(key)
                print(f"   {label:16s} {r[i]:>14s} {units[i]}")
    print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
