"""Summarise an `ncu --page source --print-source sass --csv` dump: the SASS
lines with the most warp-stall samples and the stall reasons behind them."""
import csv
import sys

def fl(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(fl(r[si]) for r in data)
agg = {}
for r in data:
    for i in stall_cols:
        agg[h[i]] = agg.get(h[i], 0) + fl(r[i])
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:24s} {100 * v / tot:5.1f}%")
top = sorted(data, key=lambda r: -fl(r[si]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    reasons = sorted(((h[i], fl(r[i])) for i in stall_cols), key=lambda x: -x[1])[:3]
    print(f"{100 * fl(r[si]) / tot:5.1f}% {r[0]:>6s} {r[1][:70]:70s} " +
          " ".join(f"{n[6:]}={100 * v / tot:.1f}" for n, v in reasons if v > 0))
